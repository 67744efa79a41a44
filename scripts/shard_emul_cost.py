"""Per-rank device time of the row-sharded inner step at config-2 size, from P emulated ranks on ONE
GPU (the ranks' kernels run one after another, so a solve's time / P is the mean per-rank compute;
collectives are device copies here, NCCL on a real box).  Compares the sharded byte floor (default)
with the sharded two-pass step (fused_path=False).  One JSON line per (P, path)."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch

import qpgen
from paper_1504_05708_b200 import Solver, solve_emulated

d = qpgen.dense_ineq_torch(16384, 8192, seed=0, shift=0.05)
args = [d[k] for k in ("Q", "q", "G", "g", "lb", "ub", "cone")]
L_in, L_d = 47588.0, 1.0 / (1.0 + 0.05 / 47539.5)
for P in (2, 4, 8):
    for fused in (True, False):
        st = torch.cuda.Stream()
        ss = [Solver(*args, rho=1.0, world_size=P, rank=r, emulate_ranks=True, stream=st.cuda_stream,
                     fused_path=fused) for r in range(P)]
        for s in ss:
            s.set_constants(L_in, L_d)
        solve_emulated(ss, "DFGM", 1, 2)                       # warm-up
        torch.cuda.synchronize()
        K, Kin = 2, 20
        t0 = time.perf_counter()
        solve_emulated(ss, "DFGM", K, Kin)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        steps = (K + 1) * Kin
        print(json.dumps(dict(P=P, path="byte_floor" if fused else "two_pass", ms_per_step_all_ranks=ms / steps,
                              ms_per_step_mean_rank=ms / steps / P)), flush=True)
        for s in ss:
            s.close()
        del ss
        torch.cuda.empty_cache()

# P = 1 on the REAL row-sharded schedule (nccl_self: one-rank NCCL communicator, graph-captured
# reduce-scatter / all-gathers) next to the plain single-GPU schedule: the schedule's own overhead
for ns in (True, False):
    s = Solver(*args, rho=1.0, nccl_self=ns)
    s.set_constants(L_in, L_d)
    s.solve("DFGM", 1, 2)
    torch.cuda.synchronize()
    K, Kin = 2, 20
    t0 = time.perf_counter()
    info = s.solve("DFGM", K, Kin)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    print(json.dumps(dict(P=1, path="byte_floor", nccl_self=ns, path_code=info["path"],
                          ms_per_step=ms / ((K + 1) * Kin))), flush=True)
    s.close()
