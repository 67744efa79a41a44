"""Warm start (duquad_set_initial) on every kernel path vs the oracle started
from the same u_bar^0 = [x0]_U and lambda^0 = mu^1 = lambda0 (-m gpu)."""
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


def _warm(prob, seed):
    rng = np.random.default_rng(seed)
    x0 = rng.uniform(-2.0, 2.0, prob.n)                         # partly outside U: projected
    lam0 = np.abs(rng.standard_normal(prob.p))                  # in K_d (>= 0 on NONPOS rows)
    return x0, lam0


def _check(torch, prob, rho, alg, K, Kin, device=False, **opts):
    from paper_1504_05708_b200 import Solver
    Qd = prob.Q.toarray() if hasattr(prob.Q, "toarray") else prob.Q
    Gd = prob.G.toarray() if hasattr(prob.G, "toarray") else prob.G
    L_in, L_d, _ = O.lipschitz_constants(Qd, Gd, rho, 0.05)
    x0, lam0 = _warm(prob, 7)
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=rho, **opts)
    s.set_constants(L_in, L_d)
    if device:
        s.set_initial(torch.from_numpy(x0).cuda(), torch.from_numpy(lam0).cuda())
    else:
        s.set_initial(x0, lam0)
    info = s.solve(alg, K, Kin)
    xl, xa, lam = s.result()
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, alg, K, Kin, L_in, L_d,
               x0=x0, lam0=lam0)
    for got, want in ((xl, r.x_last), (xa, r.x_avg), (lam, r.lam)):
        assert relerr(got, want) <= TOL, relerr(got, want)
    # reset: back to the cold start
    s.set_initial(None, None)
    s.solve(alg, K, Kin)
    xl2, _, lam2 = s.result()
    c = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, alg, K, Kin, L_in, L_d)
    assert relerr(xl2, c.x_last) <= TOL and relerr(lam2, c.lam) <= TOL
    s.close()
    return info


@pytest.mark.parametrize("alg", ["DGM", "DFGM"])
def test_warm_start_small_kernel(torch_cuda, alg):
    info = _check(torch_cuda, qpgen.dense_ineq(50, 25, seed=0), 1.0, alg, 6, 8)
    assert info["path"] == 6


def test_warm_start_two_pass_and_device_inputs(torch_cuda):
    prob = qpgen.tiny(300, 120, seed=3, kind="mixed", shift=0.2)
    info = _check(torch_cuda, prob, 1.0, "DFGM", 5, 7, device=True, small_path=False, persist_path=False)
    assert info["path"] == 0


def test_warm_start_persistent_path(torch_cuda):
    info = _check(torch_cuda, qpgen.tiny(300, 120, seed=3, kind="mixed", shift=0.2), 1.0, "DGM", 5, 7,
                  small_path=False, persist_path=True)
    assert info["path"] == 7


def test_warm_start_rho0_path(torch_cuda):
    info = _check(torch_cuda, qpgen.dense_ineq(600, 300, seed=2), 0.0, "DFGM", 4, 6, small_path=False)
    assert info["path"] == 2


@pytest.mark.parametrize("rho", [1.0, 0.0])
def test_warm_start_byte_floor(torch_cuda, rho):
    info = _check(torch_cuda, qpgen.dense_ineq(4096, 2048, seed=1, shift=0.05), rho, "DFGM", 2, 4)
    assert info["path"] in (1, 3)


def test_warm_start_csr(torch_cuda):
    info = _check(torch_cuda, qpgen.sparse_banded_eq(n=3001, p=1201, seed=4), 5.0, "DFGM", 4, 5)
    assert info["path"] == 5


def test_warm_start_batched(torch_cuda):
    """Batched (B QPs sharing Q, G): x0 is B x n and lambda0 B x p, one row per QP."""
    from paper_1504_05708_b200 import Solver
    prob = qpgen.mpc_batch(37, seed=0)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    rng = np.random.default_rng(5)
    x0 = rng.uniform(-2, 2, (37, prob.n))
    lam0 = np.abs(rng.standard_normal((37, prob.p)))
    s = Solver(prob.Q, prob.q.T.copy(), prob.G, prob.g.T.copy(), prob.lb, prob.ub, prob.cone, rho=1.0)
    s.set_constants(L_in, L_d)
    s.set_initial(x0, lam0)
    s.solve("DFGM", 4, 5)
    xl, xa, lam = s.result()
    s.close()
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, "DFGM", 4, 5, L_in, L_d,
               x0=x0.T.copy(), lam0=lam0.T.copy())
    assert relerr(xl, r.x_last.T) <= TOL and relerr(xa, r.x_avg.T) <= TOL and relerr(lam, r.lam.T) <= TOL


def test_warm_start_sharded_emulated(torch_cuda):
    """Row-sharded contexts (3 emulated ranks on one GPU) take their slices of x0 and lambda0."""
    from paper_1504_05708_b200 import Solver, solve_emulated
    import torch
    prob = qpgen.tiny(301, 97, seed=6, kind="mixed", shift=0.2)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.2)
    x0, lam0 = _warm(prob, 9)
    st = torch.cuda.Stream()
    ss = [Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0, world_size=3, rank=r,
                 emulate_ranks=True, stream=st.cuda_stream, small_path=False) for r in range(3)]
    for s in ss:
        s.set_constants(L_in, L_d)
        s.set_initial(x0, lam0)
    solve_emulated(ss, "DFGM", 5, 6)
    xl = np.concatenate([s.result()[0] for s in ss])
    lam = np.concatenate([s.result()[2] for s in ss])
    for s in ss:
        s.close()
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, "DFGM", 5, 6, L_in, L_d,
               x0=x0, lam0=lam0)
    assert relerr(xl, r.x_last) <= TOL and relerr(lam, r.lam) <= TOL


@pytest.mark.parametrize("Kin", [5, 7])
def test_warm_start_ping_pong_paths_odd_inner_count(torch_cuda, Kin):
    """rho = 0 (K3) and EQ_H ping-pong y between two replicas; odd K_in makes the DFOM step read
    the second one: cold and warm starts must still match the oracle."""
    info = _check(torch_cuda, qpgen.dense_ineq(600, 300, seed=2), 0.0, "DFGM", 4, Kin, small_path=False)
    assert info["path"] == 2
    info = _check(torch_cuda, qpgen.tiny(500, 150, seed=14, kind="eq"), 1.0, "DGM", 3, Kin, small_path=False)
    assert info["path"] == 8
