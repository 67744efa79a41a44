"""Equality-QP precomputation (NEXT-3) at config-2 size: n = 16384, p = 8192, every row an equality
(the config-2 recipe with the cone set to ZERO; x0 = the generator's interior point, g = -G x0), DFGM
rho = 1.  Times the inner step with eq_precompute on (H = Q + rho G'G, path eq_h_floor) and off
(the generic byte-floor step), and the one-time setup (H via cuBLAS DGEMM).  One JSON line each."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch

import qpgen
from paper_1504_05708_b200 import Solver

n, p = 16384, 8192
d = qpgen.dense_ineq_torch(n, p, seed=0)
d["cone"].zero_()                                   # all rows equalities (K = {0})
st = torch.cuda.Stream()
for eq in (True, False):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = Solver(d["Q"], d["q"], d["G"], d["g"], d["lb"], d["ub"], d["cone"], rho=1.0, lambda_min_lb=0.05,
               stream=st.cuda_stream, eq_precompute=eq)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    s.lipschitz(iters=30, safety=1e-3)
    s.solve("DFGM", 1, 5)                            # warm-up
    K, Kin = 4, 50
    info = s.solve("DFGM", K, Kin)
    ms = info["ms_device"]
    print(json.dumps(dict(eq_precompute=eq, path=info["path"], setup_s=t_setup, ms_per_solve=ms,
                          us_per_inner_step=ms * 1e3 / ((K + 1) * Kin),
                          inner_iters_per_s=(K + 1) * Kin / (ms / 1e3))), flush=True)
    s.close()
