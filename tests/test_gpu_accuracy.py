"""North-star accuracy criterion (-m gpu): at the configured iteration counts, the GPU solution
satisfies |F(x) - F*| <= 1e-3 (1 + |F*|) and ||dist_K(G x + g)|| <= 1e-3 for the last iterate and the
primal average, with F* from a long oracle run (configs 0, 1 and, with 500 inner steps, an
8-QP subset of config 3)."""
import numpy as np
import pytest

import qpgen
from oracle import dfom as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _fstar(prob, rho, L_in, L_d, K, Kin):
    """F* of a long oracle DFGM run (its last iterate), and its infeasibility."""
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, O.DFGM, K, Kin, L_in, L_d)
    x = r.x_last
    return O.objective(prob.Q, prob.q, x), O.dist_K(prob.G @ x + prob.g, prob.cone)


def _criteria(prob, x, Fs):
    F = O.objective(prob.Q, prob.q, x)
    d = O.dist_K(prob.G @ x + prob.g, prob.cone)
    return np.abs(F - Fs) <= 1e-3 * (1 + np.abs(Fs)), d <= 1e-3


@pytest.mark.parametrize("cfg", [0, 1])
def test_dense_configs_meet_the_accuracy_criterion(torch_cuda, cfg):
    from paper_1504_05708_b200 import Solver
    c = qpgen.CONFIGS[cfg]
    prob = qpgen.dense_ineq(c["n"], c["p"], seed=0, shift=c["shift"])
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, c["rho"], c["lambda_min_lb"])
    Fs, ds = _fstar(prob, c["rho"], L_in, L_d, *((2000, 100) if cfg == 0 else (200, 100)))
    assert ds <= 1e-6
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=c["rho"])
    s.set_constants(L_in, L_d)
    s.solve(c["alg"], c["outer"], c["inner"])
    xl, xa, _ = s.result()
    s.close()
    for x in (xl, xa):
        okF, okd = _criteria(prob, x, Fs)
        assert okF and okd, (O.objective(prob.Q, prob.q, x), Fs, O.dist_K(prob.G @ x + prob.g, prob.cone))


def test_batched_config3_subset_meets_the_accuracy_criterion(torch_cuda):
    """Config 3's MPC Hessian is badly conditioned (L_in ~ 6e5 at rho = 1, lambda_min >= 0.1): the
    configured 50 x 20 counts match the oracle (test_gpu_batched) but are far from the 1e-3
    criterion (|F - F*| ~ 0.24 relative); with 500 inner steps per solve it is met.
    First 8 QPs of the batch; F* from a 50 x 1500 oracle run (stable to 1e-15 against 60 x 6000)."""
    from paper_1504_05708_b200 import Solver
    c = qpgen.CONFIGS[3]
    prob = qpgen.mpc_batch(8, seed=0)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, c["rho"], c["lambda_min_lb"])
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, c["rho"], O.DFGM, 50, 1500, L_in, L_d)
    Fs = O.objective(prob.Q, prob.q, r.x_last)                       # per QP
    s = Solver(prob.Q, prob.q.T.copy(), prob.G, prob.g.T.copy(), prob.lb, prob.ub, prob.cone, rho=c["rho"])
    s.set_constants(L_in, L_d)
    s.solve(c["alg"], c["outer"], 500)
    xl, xa, _ = s.result()
    s.close()
    for X in (xl, xa):
        x = X.T                                                       # n x B, one column per QP
        okF, okd = _criteria(prob, x, Fs)
        assert np.all(okF) and np.all(okd)
