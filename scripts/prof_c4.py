"""Config 4 solve-mode launches only (constants injected, no Lanczos) for ncu captures."""
import sys
sys.path.insert(0, ".")
import qpgen
from paper_1504_05708_b200 import Solver
prob = qpgen.sparse_banded_eq()
s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=5.0, lambda_min_lb=0.5, use_graphs=False)
s.set_constants(240.4, 0.1996)
s.solve("DFGM", 1, 3)
print("ok")
