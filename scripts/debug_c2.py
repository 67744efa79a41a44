import sys, numpy as np, torch
sys.path.insert(0, '.')
import qpgen
from oracle import dfom as O
from paper_1504_05708_b200 import Solver
def rel(a, b): return float(np.max(np.abs(a-b))/(1+np.max(np.abs(b))))
for n, p in [(2048, 1024), (8192, 4096), (16384, 8192)]:
    d = qpgen.dense_ineq_torch(n, p, seed=0, shift=0.05)
    s = Solver(d["Q"], d["q"], d["G"], d["g"], d["lb"], d["ub"], d["cone"], rho=1.0, lambda_min_lb=0.05)
    L_in, L_d, nG2 = s.lipschitz(iters=60, safety=1e-3)
    h = {k: v.cpu().numpy() for k, v in d.items()}
    for (K, Kin) in [(1, 1), (1, 2), (2, 2)]:
        s.solve("DFGM", K, Kin)
        xl, xa, lam = s.result()
        r = O.dfom(h["Q"], h["q"], h["G"], h["g"], h["lb"], h["ub"], h["cone"], 1.0, O.DFGM, K, Kin, L_in, L_d)
        print(n, p, K, Kin, "L", L_in, L_d, "err", rel(xl, r.x_last), rel(xa, r.x_avg), rel(lam, r.lam), flush=True)
    # single GEMV check through residuals: F of x_last
    F, dist, lag = s.residuals("last")
    print("F", F, O.objective(h["Q"], h["q"], xl), "dist", dist, O.dist_K(h["G"] @ xl + h["g"], h["cone"]), flush=True)
    s.close(); del d, h
