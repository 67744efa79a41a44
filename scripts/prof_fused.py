"""One config-2 solve (1 x 2 inner steps, no graphs) for ncu captures of the fused kernels.
PROF_RHO (default 1) selects rho; rho = 0 runs the Q-only stream (K3 path)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import qpgen
from paper_1504_05708_b200 import Solver

rho = float(os.environ.get("PROF_RHO", "1"))
d = qpgen.dense_ineq_torch(16384, 8192, seed=0, shift=0.05)
st = torch.cuda.Stream()
s = Solver(d["Q"], d["q"], d["G"], d["g"], d["lb"], d["ub"], d["cone"], rho=rho, lambda_min_lb=0.05,
           stream=st.cuda_stream, use_graphs=False)
s.set_constants(47588.0, 1.0)
s.solve("DFGM", 1, 2)
torch.cuda.synchronize()
print("ok")
