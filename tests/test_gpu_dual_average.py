"""DGM dual-averaging final point (options.dual_average) on every
kernel path vs the oracle's dfom(dual_average=True) (-m gpu): lambda^K := [lam_hat + grad_bar
d(lam_hat)/(2 L_d)]_{K_d}, lam_hat the average of lambda^0..lambda^K, x_last = u_bar(lambda^K)."""
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


def _check(prob, rho, K, Kin, lmin=0.1, **opts):
    from paper_1504_05708_b200 import Solver
    Qd = prob.Q.toarray() if hasattr(prob.Q, "toarray") else prob.Q
    Gd = prob.G.toarray() if hasattr(prob.G, "toarray") else prob.G
    L_in, L_d, _ = O.lipschitz_constants(Qd, Gd, rho, lmin)
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=rho, dual_average=True, **opts)
    s.set_constants(L_in, L_d)
    info = s.solve("DGM", K, Kin)
    xl, xa, lam = s.result()
    s.close()
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, O.DGM, K, Kin, L_in, L_d,
               dual_average=True)
    for got, want in ((xl, r.x_last), (xa, r.x_avg), (lam, r.lam)):
        assert relerr(got, want) <= TOL, relerr(got, want)
    plain = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, O.DGM, K, Kin, L_in, L_d)
    assert relerr(lam, plain.lam) > 1e-6            # the averaged point is a different point
    return info


def test_two_pass_mixed_cones(torch_cuda):
    info = _check(qpgen.tiny(300, 120, seed=3, kind="mixed", shift=0.2), 1.0, 6, 7, 0.2, small_path=False)
    assert info["path"] == 0 and info["inner_iters_total"] == (6 + 2) * 7


def test_small_problem_defers_from_the_single_cta_kernel(torch_cuda):
    info = _check(qpgen.dense_ineq(50, 25, seed=0), 1.0, 8, 10)
    assert info["path"] == 0


def test_rho0_path(torch_cuda):
    info = _check(qpgen.dense_ineq(600, 300, seed=2), 0.0, 4, 6, small_path=False)
    assert info["path"] == 2


@pytest.mark.parametrize("rho", [1.0, 0.0])
def test_byte_floor(torch_cuda, rho):
    info = _check(qpgen.dense_ineq(4096, 2048, seed=1, shift=0.05), rho, 2, 4, 0.05)
    assert info["path"] in (1, 3)


def test_csr(torch_cuda):
    info = _check(qpgen.sparse_banded_eq(n=3001, p=1201, seed=4), 5.0, 4, 5, 0.5)
    assert info["path"] == 5


def test_batched(torch_cuda):
    from paper_1504_05708_b200 import Solver
    prob = qpgen.mpc_batch(37, seed=0)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    s = Solver(prob.Q, prob.q.T.copy(), prob.G, prob.g.T.copy(), prob.lb, prob.ub, prob.cone, rho=1.0,
               dual_average=True)
    s.set_constants(L_in, L_d)
    s.solve("DGM", 4, 5)
    xl, xa, lam = s.result()
    s.close()
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, O.DGM, 4, 5, L_in, L_d,
               dual_average=True)
    assert relerr(xl, r.x_last.T) <= TOL and relerr(xa, r.x_avg.T) <= TOL and relerr(lam, r.lam.T) <= TOL


def test_sharded_emulated(torch_cuda):
    from paper_1504_05708_b200 import Solver, solve_emulated
    import torch
    prob = qpgen.tiny(301, 97, seed=6, kind="mixed", shift=0.2)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.2)
    st = torch.cuda.Stream()
    ss = [Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0, world_size=3, rank=r,
                 emulate_ranks=True, stream=st.cuda_stream, small_path=False, dual_average=True) for r in range(3)]
    for s in ss:
        s.set_constants(L_in, L_d)
    solve_emulated(ss, "DGM", 5, 6)
    xl = np.concatenate([s.result()[0] for s in ss])
    lam = np.concatenate([s.result()[2] for s in ss])
    for s in ss:
        s.close()
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, O.DGM, 5, 6, L_in, L_d,
               dual_average=True)
    assert relerr(xl, r.x_last) <= TOL and relerr(lam, r.lam) <= TOL


def test_rejected_with_dfgm_and_eps_mode(torch_cuda):
    from paper_1504_05708_b200 import Solver, DuquadError
    prob = qpgen.dense_ineq(50, 25, seed=0)
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0, dual_average=True)
    s.set_constants(100.0, 1.0)
    with pytest.raises(DuquadError):
        s.solve("DFGM", 2, 3)
    with pytest.raises(DuquadError):
        s.solve_eps("DGM", 2, 10, 1e-6, 0.1)
    s.solve("DGM", 2, 3)      # the context is still usable
    s.close()
