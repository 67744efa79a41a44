"""Config-0 solve through the single-CTA whole-solve kernel (K4), for ncu captures."""
import sys
sys.path.insert(0, ".")
import qpgen
from oracle import dfom as O
from paper_1504_05708_b200 import Solver
prob = qpgen.dense_ineq(50, 25, seed=0)
L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0)
s.set_constants(L_in, L_d)
info = s.solve("DFGM", 40, 50)
print("ok", info["ms_device"], info["path"])
