"""Per-CTA start / end of one byte-floor stream launch (config 2), from a DQ_TRACE_ROLE build of the
library (scripts/gpu_role.sh): which role's CTAs finish last, and by how much."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import qpgen  # noqa: E402
from paper_1504_05708_b200 import Solver, _lib  # noqa: E402

torch.cuda.set_device(0)
d = qpgen.dense_ineq_torch(16384, 8192, seed=0, shift=0.05, device="cuda:0")
s = Solver(d["Q"], d["q"], d["G"], d["g"], d["lb"], d["ub"], d["cone"], rho=1.0, lambda_min_lb=0.05)
s.lipschitz(iters=60, safety=1e-3)
s.solve("DFGM", 100, 100)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 320)()
rc = _lib.lib().duquad_debug_role_trace(buf, 320)
nq = int(os.environ.get("DUQUAD_FUSED_NQ", "66"))
t0 = min(buf[2 * c] for c in range(148))
rows = [(c, (buf[2 * c] - t0) / 1e3, (buf[2 * c + 1] - t0) / 1e3) for c in range(148)]
q = [r[2] for r in rows[:nq]]
g = [r[2] for r in rows[nq:]]
out = {"rc": rc, "nq": nq, "start_max_us": max(r[1] for r in rows),
       "q_end_us": [min(q), sorted(q)[len(q) // 2], max(q)], "g_end_us": [min(g), sorted(g)[len(g) // 2], max(g)],
       "ends": [round(r[2], 1) for r in rows]}
print(json.dumps(out))
