import os, sys
sys.path.insert(0, '.')
import numpy as np
import qpgen
from oracle import dfom as O
from paper_1504_05708_b200 import Solver
prob = qpgen.sparse_banded_eq(n=3001, p=1201, seed=4)
Qd, Gd = prob.Q.toarray(), prob.G.toarray()
L_in, L_d, _ = O.lipschitz_constants(Qd, Gd, 5.0, 0.05)
rng = np.random.default_rng(7)
x0 = rng.uniform(-2.0, 2.0, prob.n); lam0 = np.abs(rng.standard_normal(prob.p))
def rel(a, b): return float(np.max(np.abs(a - b)) / (1 + np.max(np.abs(b))))
for dia in ("1", "0"):
    os.environ["DUQUAD_DIA"] = dia
    for warm in (False, True):
        for graphs in (True, False):
            s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=5.0, use_graphs=graphs)
            s.set_constants(L_in, L_d)
            if warm: s.set_initial(x0, lam0)
            info = s.solve("DFGM", 4, 5)
            xl, xa, lam = s.result()
            r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 5.0, "DFGM", 4, 5, L_in, L_d,
                       x0=x0 if warm else None, lam0=lam0 if warm else None)
            print("dia", dia, "warm", warm, "graphs", graphs, "kern", info["sparse_kernels"], "err", rel(xl, r.x_last), rel(lam, r.lam), flush=True)
            s.close()
