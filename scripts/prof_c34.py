"""Config 3 (batched DMMA) and config 4 (CSR) prefixes for ncu captures: PROF_CFG=3|4."""
import os
import sys
sys.path.insert(0, ".")
import qpgen
from paper_1504_05708_b200 import Solver
cfg = int(os.environ.get("PROF_CFG", "3"))
if cfg == 3:
    prob = qpgen.mpc_batch(8192, seed=0)
    s = Solver(prob.Q, prob.q.T.copy(), prob.G, prob.g.T.copy(), prob.lb, prob.ub, prob.cone, rho=1.0,
               lambda_min_lb=0.1, use_graphs=False)
else:
    prob = qpgen.sparse_banded_eq()
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=5.0, lambda_min_lb=0.5,
               use_graphs=False)
s.lipschitz(iters=40, safety=1e-3)
s.solve("DFGM", 1, 3)
print("ok")
