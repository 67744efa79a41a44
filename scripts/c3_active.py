"""Config 3 (SURVEY §8(d) note): fraction of active constraint rows and box faces at the reference
solution (DFGM rho = 1, 50 x 500 -- the counts that meet the 1e-3 accuracy criterion, see
tests/test_gpu_accuracy.py) over all 8192 QPs."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np

import qpgen
from paper_1504_05708_b200 import Solver

prob = qpgen.mpc_batch(8192, seed=0)
s = Solver(prob.Q, prob.q.T.copy(), prob.G, prob.g.T.copy(), prob.lb, prob.ub, prob.cone, rho=1.0,
           lambda_min_lb=0.1)
s.lipschitz(iters=80, safety=1e-3)
info = s.solve("DFGM", 50, 500)
xl, xa, lam = s.result()
s.close()
X = xl.T                                              # n x B
r = prob.G @ X + prob.g                               # p x B, K = R^p_- (all rows NONPOS)
act = r > -1e-6
box = (np.abs(X - prob.lb[:, None]) < 1e-9) | (np.abs(X - prob.ub[:, None]) < 1e-9)
print(json.dumps(dict(config=3, solve="DFGM rho=1 50x500", ms=info["ms_device"],
                      active_constraint_rows_frac=float(act.mean()), qps_with_an_active_row=float(act.any(0).mean()),
                      box_active_frac=float(box.mean()), qps_with_an_active_bound=float(box.any(0).mean()),
                      max_violation=float(np.maximum(r, 0).max()), nonzero_multipliers_frac=float((lam > 1e-9).mean()))))
