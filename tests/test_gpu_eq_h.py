"""Equality-QP precomputation (options.eq_precompute) vs the
oracle (-m gpu): with every row an equality, grad L_rho = (Q + rho G'G) u + q + G'(mu + rho g), so
H = Q + rho G'G is formed once and each inner step streams H alone (path EQ_H, or EQ_H_FLOOR with
the byte-floor kernel over H's upper triangle).  The oracle runs the generic DFOM."""
import numpy as np
import pytest

import qpgen
from oracle import dfom as O

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def relerr(got, want):
    got, want = np.asarray(got, float), np.asarray(want, float)
    return float(np.max(np.abs(got - want)) / (1.0 + np.max(np.abs(want)))) if want.size else 0.0


def _run(prob, rho, alg, K, Kin, lmin=0.2, **kw):
    from paper_1504_05708_b200 import Solver
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, rho, lmin)
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=rho, **kw)
    s.set_constants(L_in, L_d)
    info = s.solve(alg, K, Kin)
    out = s.result()
    s.close()
    return info, out, (L_in, L_d)


@pytest.mark.parametrize("alg", ["DGM", "DFGM"])
def test_eq_h_two_pass_size(torch_cuda, alg):
    prob = qpgen.tiny(600, 200, seed=11, kind="eq")
    info, (xl, xa, lam), (L_in, L_d) = _run(prob, 1.0, alg, 5, 8, small_path=False)
    assert info["path"] == 8
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, alg, 5, 8, L_in, L_d)
    for got, want in ((xl, r.x_last), (xa, r.x_avg), (lam, r.lam)):
        assert relerr(got, want) <= TOL, relerr(got, want)
    # the generic inner step on the same problem agrees
    info0, (xl0, _, lam0), _ = _run(prob, 1.0, alg, 5, 8, small_path=False, eq_precompute=False)
    assert info0["path"] == 0 and relerr(xl0, xl) <= TOL and relerr(lam0, lam) <= TOL


def test_eq_h_byte_floor(torch_cuda):
    prob = qpgen.tiny(4096, 1024, seed=12, kind="eq")
    info, (xl, xa, lam), (L_in, L_d) = _run(prob, 2.0, "DFGM", 2, 4)
    assert info["path"] == 9
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 2.0, "DFGM", 2, 4, L_in, L_d)
    for got, want in ((xl, r.x_last), (xa, r.x_avg), (lam, r.lam)):
        assert relerr(got, want) <= TOL, relerr(got, want)


def test_eq_h_cone_all_and_mixed_rows(torch_cuda):
    from paper_1504_05708_b200 import Solver, _lib
    prob = qpgen.tiny(300, 90, seed=13, kind="eq")
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.2)
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, None, rho=1.0, cone_all=_lib.CONE_ZERO,
               small_path=False)
    s.set_constants(L_in, L_d)
    assert s.solve("DFGM", 3, 5)["path"] == 8
    xl, _, lam = s.result()
    s.close()
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, "DFGM", 3, 5, L_in, L_d)
    assert relerr(xl, r.x_last) <= TOL and relerr(lam, r.lam) <= TOL
    mixed = qpgen.tiny(300, 90, seed=13, kind="mixed")
    info, _, _ = _run(mixed, 1.0, "DFGM", 2, 3, small_path=False)
    assert info["path"] == 0                                   # an inequality row: no H path


def test_eq_h_with_dual_average_warm_start_and_eps_mode(torch_cuda):
    from paper_1504_05708_b200 import Solver
    prob = qpgen.tiny(500, 150, seed=14, kind="eq")
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.2)
    # DGM dual averaging on the H path
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0, small_path=False,
               dual_average=True)
    s.set_constants(L_in, L_d)
    assert s.solve("DGM", 4, 6)["path"] == 8
    xl, _, lam = s.result()
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, "DGM", 4, 6, L_in, L_d,
               dual_average=True)
    assert relerr(xl, r.x_last) <= TOL and relerr(lam, r.lam) <= TOL
    s.close()
    # warm start
    rng = np.random.default_rng(3)
    x0, lam0 = rng.uniform(-2, 2, 500), rng.standard_normal(150)
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0, small_path=False)
    s.set_constants(L_in, L_d)
    s.set_initial(x0, lam0)
    s.solve("DFGM", 3, 5)
    xl, _, lam = s.result()
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, "DFGM", 3, 5, L_in, L_d,
               x0=x0, lam0=lam0)
    assert relerr(xl, r.x_last) <= TOL and relerr(lam, r.lam) <= TOL
    # eps_in mode: the GPU's per-solve counts replayed by the oracle
    s.set_initial(None, None)
    info = s.solve_eps("DFGM", 3, 300, 1e-6, 0.2)
    assert info["path"] == 8
    xl, _, lam = s.result()
    s.close()
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, "DFGM", 3, info["inner_counts"],
               L_in, L_d)
    assert relerr(xl, r.x_last) <= TOL and relerr(lam, r.lam) <= TOL
