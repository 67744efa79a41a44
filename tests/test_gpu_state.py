"""State export / resume (duquad_get_state / duquad_set_state) (-m gpu):
solve(K1) + get_state + set_state + solve(K2) is bitwise solve(K1 + K2) on every streaming path, and
the exported state is the oracle's DFOM state after K outer iterations."""
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


def _mk(prob, rho, L, batched=False, **kw):
    from paper_1504_05708_b200 import Solver
    q, g = (prob.q.T.copy(), prob.g.T.copy()) if batched else (prob.q, prob.g)
    s = Solver(prob.Q, q, prob.G, g, prob.lb, prob.ub, prob.cone, rho=rho, checkpoint=True, **kw)
    s.set_constants(*L)
    return s


def _resume_bitwise(prob, rho, alg, K1, K2, Kin, lmin=0.2, batched=False, fresh=False, **kw):
    Qd = prob.Q.toarray() if hasattr(prob.Q, "toarray") else prob.Q
    Gd = prob.G.toarray() if hasattr(prob.G, "toarray") else prob.G
    L = O.lipschitz_constants(Qd, Gd, rho, lmin)[:2]
    s = _mk(prob, rho, L, batched, **kw)
    info = s.solve(alg, K1 + K2, Kin)
    full = s.result()
    s.solve(alg, K1, Kin)
    st = s.get_state()
    assert st["outer_done"] == K1
    t = _mk(prob, rho, L, batched, **kw) if fresh else s
    t.set_state(st)
    t.solve(alg, K2, Kin)
    part = t.result()
    st2 = t.get_state()
    assert st2["outer_done"] == K1 + K2
    for a, b in zip(full, part):
        assert np.array_equal(a, b), np.max(np.abs(a - b))
    s.close()
    if fresh:
        t.close()
    return info


@pytest.mark.parametrize("alg", ["DGM", "DFGM"])
def test_resume_two_pass_bitwise(torch_cuda, alg):
    info = _resume_bitwise(qpgen.tiny(300, 120, seed=3, kind="mixed", shift=0.2), 1.0, alg, 3, 4, 6,
                           small_path=False)
    assert info["path"] == 0


def test_resume_small_problem_defers_from_k4_and_fresh_context(torch_cuda):
    info = _resume_bitwise(qpgen.dense_ineq(50, 25, seed=0), 1.0, "DFGM", 5, 2, 8, lmin=0.1, fresh=True)
    assert info["path"] == 0


def test_resume_byte_floor_rho0_eq_h_csr(torch_cuda):
    assert _resume_bitwise(qpgen.dense_ineq(4096, 2048, seed=1, shift=0.05), 1.0, "DFGM", 1, 2, 3,
                           lmin=0.05)["path"] == 1
    assert _resume_bitwise(qpgen.dense_ineq(600, 300, seed=2), 0.0, "DFGM", 2, 2, 4, lmin=0.1,
                           small_path=False)["path"] == 2
    assert _resume_bitwise(qpgen.tiny(500, 150, seed=14, kind="eq"), 1.0, "DFGM", 2, 3, 4,
                           small_path=False)["path"] == 8
    assert _resume_bitwise(qpgen.sparse_banded_eq(n=3001, p=1201, seed=4), 5.0, "DFGM", 2, 2, 4,
                           lmin=0.5)["path"] == 5


@pytest.mark.parametrize("fresh", [False, True])
def test_resume_odd_inner_count(torch_cuda, fresh):
    """Odd K_in on the paths that ping-pong y between two replicas (rho = 0 K3, its Q-only byte floor,
    EQ_H): the DFOM step after a resume reads the replica the previous inner solve finished in,
    Y[K_in % 2], so both replicas must restart at u_bar^{j0} (regression: only Y[0] was)."""
    assert _resume_bitwise(qpgen.dense_ineq(600, 300, seed=2), 0.0, "DFGM", 2, 3, 5, lmin=0.1,
                           small_path=False, fresh=fresh)["path"] == 2
    assert _resume_bitwise(qpgen.tiny(500, 150, seed=14, kind="eq"), 1.0, "DFGM", 2, 3, 3,
                           small_path=False, fresh=fresh)["path"] == 8
    assert _resume_bitwise(qpgen.dense_ineq(4096, 2048, seed=1, shift=0.05), 0.0, "DFGM", 1, 2, 3,
                           lmin=0.05, fresh=fresh)["path"] == 3


def test_resume_odd_inner_count_sharded_rho0(torch_cuda):
    """The same on 3 emulated row-sharded ranks at rho = 0: the second replica is re-gathered."""
    from paper_1504_05708_b200 import Solver, solve_emulated
    import torch
    prob = qpgen.dense_ineq(301, 97, seed=2, shift=0.1)
    L = O.lipschitz_constants(prob.Q, prob.G, 0.0, 0.1)[:2]
    st = torch.cuda.Stream()

    def group():
        ss = [Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=0.0, world_size=3, rank=r,
                     emulate_ranks=True, stream=st.cuda_stream, small_path=False, checkpoint=True) for r in range(3)]
        for s in ss:
            s.set_constants(*L)
        return ss

    a = group()
    solve_emulated(a, "DFGM", 5, 5)
    full = [np.concatenate([s.result()[i] for s in a]) for i in range(3)]
    solve_emulated(a, "DFGM", 2, 5)
    states = [s.get_state() for s in a]
    b = group()
    for s, stt in zip(b, states):
        s.set_state(stt)
    solve_emulated(b, "DFGM", 3, 5)
    part = [np.concatenate([s.result()[i] for s in b]) for i in range(3)]
    for s in a + b:
        s.close()
    for x, y in zip(full, part):
        assert np.array_equal(x, y), np.max(np.abs(x - y))


def test_resume_batched(torch_cuda):
    _resume_bitwise(qpgen.mpc_batch(37, seed=0), 1.0, "DFGM", 2, 3, 5, lmin=0.1, batched=True)


@pytest.mark.parametrize("alg", ["DGM", "DFGM"])
def test_state_is_the_oracle_state_after_K(torch_cuda, alg):
    prob = qpgen.tiny(300, 120, seed=3, kind="mixed", shift=0.2)
    L = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.2)[:2]
    s = _mk(prob, 1.0, L, small_path=False)
    K, Kin = 4, 6
    s.solve(alg, K, Kin)
    st = s.get_state()
    s.close()
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, alg, K, Kin, *L, keep_trace=True)
    assert relerr(st["x"], r.trace_u[K - 1]) <= TOL                 # u_bar^K
    assert relerr(st["mu"], r.trace_mu[K - 1]) <= TOL               # mu^K
    assert relerr(st["lam_prev"], r.trace_lam[K - 2]) <= TOL        # lambda^{K-1}
    assert relerr(st["x_avg"], r.x_avg) <= TOL
    assert st["S"] == pytest.approx(r.S, rel=1e-15)


def test_state_errors(torch_cuda):
    from paper_1504_05708_b200 import Solver, DuquadError
    prob = qpgen.dense_ineq(50, 25, seed=0)
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0)
    s.set_constants(100.0, 1.0)
    s.solve("DFGM", 2, 3)
    with pytest.raises(DuquadError):
        s.get_state()                                   # no checkpoint option
    bad = dict(x=np.zeros(50), mu=np.zeros(25), lam_prev=np.zeros(25), x_avg=np.zeros(50), outer_done=0, S=1.0)
    with pytest.raises(DuquadError):
        s.set_state(bad)
    s.close()
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0, checkpoint=True,
               dual_average=True)
    s.set_constants(100.0, 1.0)
    with pytest.raises(DuquadError):
        s.solve("DGM", 2, 3)                            # checkpoint + dual averaging: not combined
    s.close()


@pytest.mark.parametrize("n,p", [(301, 97), (4100, 1500)])
def test_resume_row_sharded_emulated(torch_cuda, n, p):
    """Row-sharded (3 emulated ranks; two-pass at n = 301, the sharded byte floor at n = 4100): each
    rank exports and re-imports its own slices; the continuation is bitwise the uninterrupted solve."""
    from paper_1504_05708_b200 import Solver, solve_emulated
    import torch
    prob = qpgen.dense_ineq(n, p, seed=2, shift=0.1)
    L = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)[:2]
    st = torch.cuda.Stream()

    def group():
        ss = [Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0, world_size=3, rank=r,
                     emulate_ranks=True, stream=st.cuda_stream, small_path=False, checkpoint=True) for r in range(3)]
        for s in ss:
            s.set_constants(*L)
        return ss

    a = group()
    solve_emulated(a, "DFGM", 5, 4)
    full = [np.concatenate([s.result()[i] for s in a]) for i in range(3)]
    solve_emulated(a, "DFGM", 2, 4)
    states = [s.get_state() for s in a]
    b = group()
    for s, stt in zip(b, states):
        s.set_state(stt)
    solve_emulated(b, "DFGM", 3, 4)
    part = [np.concatenate([s.result()[i] for s in b]) for i in range(3)]
    for s in a + b:
        s.close()
    for x, y in zip(full, part):
        assert np.array_equal(x, y), np.max(np.abs(x - y))
