"""eps_in-driven inner stopping (duquad_solve_eps) vs the oracle (-m gpu).

The stop decisions are floating-point decisions taken on the device (fixed-order sum of
(y - x+)^2) and in the oracle (NumPy norm); near the threshold they could differ in the last
bit, so parity is checked the way the task prescribes for such decisions: the oracle replays the
GPU's per-solve step counts (iterates must agree to 1e-9), and every GPU decision is checked
against the oracle's gradient-map values at the same iterate (stop => L||y-x+|| <= thr,
continue => > thr, up to 1e-8 relative)."""
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


def _run(prob, rho, alg, K, kmax, eps_in, sigma_L, L_in, L_d, **kw):
    from paper_1504_05708_b200 import Solver
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=rho, **kw)
    s.set_constants(L_in, L_d)
    info = s.solve_eps(alg, K, kmax, eps_in, sigma_L)
    xl, xa, lam = s.result()
    s.close()
    return info, xl, xa, lam


def _check(prob, rho, alg, K, kmax, eps_in, sigma_L, L_in, L_d, info, xl, xa, lam):
    counts, conv = info["inner_counts"], info["converged"]
    assert len(counts) == K + 1 and info["inner_iters_total"] == sum(counts)
    assert all(1 <= c <= kmax for c in counts)
    assert any(conv), "no inner solve met the eps_in test: pick a larger eps_in"
    assert info["capped"] == (not all(conv))
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, alg, K, counts, L_in, L_d,
               record_gm=True)
    for got, want in ((xl, r.x_last), (xa, r.x_avg), (lam, r.lam)):
        assert relerr(got, want) <= TOL, relerr(got, want)
    thr = np.sqrt(2.0 * sigma_L * eps_in)
    for j, (c, cv) in enumerate(zip(counts, conv)):
        gm = r.gm[j]
        assert len(gm) == c
        assert all(v > thr * (1 - 1e-8) for v in gm[:-1]), (j, gm, thr)   # did not stop too late
        if cv:
            assert gm[-1] <= thr * (1 + 1e-8), (j, gm[-1], thr)             # stopped legitimately
        else:
            assert c == kmax and gm[-1] > thr * (1 - 1e-8)


@pytest.mark.parametrize("rho,alg", [(1.0, "DFGM"), (1.0, "DGM"), (0.0, "DFGM"), (10.0, "DFGM")])
def test_eps_mode_dense_two_pass(torch_cuda, rho, alg):
    prob = qpgen.dense_ineq(50, 25, seed=0)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, rho, 0.1)
    eps_in, sigma_L, K, kmax = 1e-7, 0.1, 12, 400
    info, xl, xa, lam = _run(prob, rho, alg, K, kmax, eps_in, sigma_L, L_in, L_d)
    _check(prob, rho, alg, K, kmax, eps_in, sigma_L, L_in, L_d, info, xl, xa, lam)
    assert len(set(info["inner_counts"])) > 1      # adaptive: the counts differ between solves


def test_eps_mode_mixed_cones_ragged(torch_cuda):
    prob = qpgen.tiny(37, 13, seed=5, kind="mixed", shift=0.2)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 2.0, 0.2)
    info, xl, xa, lam = _run(prob, 2.0, "DFGM", 8, 300, 1e-8, 0.2, L_in, L_d)
    _check(prob, 2.0, "DFGM", 8, 300, 1e-8, 0.2, L_in, L_d, info, xl, xa, lam)


def test_eps_mode_cap_reports_emaxiter(torch_cuda):
    prob = qpgen.dense_ineq(50, 25, seed=0)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    from paper_1504_05708_b200 import Solver
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0)
    s.set_constants(L_in, L_d)
    info = s.solve_eps("DFGM", 4, 3, 1e-14, 0.1)   # unreachable accuracy: every solve is capped
    assert info["capped"] and info["inner_counts"] == [3] * 5 and not any(info["converged"])
    xl, xa, lam = s.result()
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, "DFGM", 4, 3, L_in, L_d)
    assert relerr(xl, r.x_last) <= TOL and relerr(lam, r.lam) <= TOL
    # a plain fixed-count solve on the same context afterwards is unaffected
    s.solve("DFGM", 4, 3)
    xl2, _, _ = s.result()
    assert relerr(xl2, r.x_last) <= TOL
    s.close()


@pytest.mark.parametrize("rho", [1.0, 0.0])
def test_eps_mode_byte_floor_path(torch_cuda, rho):
    """n >= 4096: the byte-floor kernels (k_fused_stream / k_fused_epi), incl. the rho = 0 Q-only one."""
    prob = qpgen.dense_ineq(4096, 2048, seed=1, shift=0.05)
    if rho > 0:   # a better-conditioned inner problem (L_in ~ 31), so inner solves converge in < 80 steps
        prob.G *= 0.05
        prob.g *= 0.05
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, rho, 0.05)
    eps_in, sigma_L, K, kmax = 1e-2, 0.05, 3, 80
    info, xl, xa, lam = _run(prob, rho, "DFGM", K, kmax, eps_in, sigma_L, L_in, L_d)
    assert info["path"] in (1, 3)
    _check(prob, rho, "DFGM", K, kmax, eps_in, sigma_L, L_in, L_d, info, xl, xa, lam)


def test_eps_mode_rho0_q_only_path(torch_cuda):
    prob = qpgen.dense_ineq(600, 300, seed=2, shift=0.1)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 0.0, 0.1)
    info, xl, xa, lam = _run(prob, 0.0, "DFGM", 6, 200, 1e-7, 0.1, L_in, L_d, small_path=False)
    assert info["path"] == 2
    _check(prob, 0.0, "DFGM", 6, 200, 1e-7, 0.1, L_in, L_d, info, xl, xa, lam)


def test_eps_mode_pass_accounting_matches_fixed_counts(torch_cuda):
    """The matvec accounting identity (SPEC.md:558, :604 item 12): an eps_in-mode solve reports the
    passes a fixed-count solve with the same per-solve step counts reports -- 2 per inner step on the
    two-pass path; on the Q-only (rho = 0) path 1 per inner step + 2 per inner solve (G u_bar, G' mu)."""
    from paper_1504_05708_b200 import Solver
    for rho, kw in ((0.0, dict(small_path=False)), (1.0, dict(small_path=False, fused_path=False))):
        prob = qpgen.dense_ineq(600, 300, seed=2, shift=0.1)
        L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, rho, 0.1)
        s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=rho, **kw)
        s.set_constants(L_in, L_d)
        K, kmax = 4, 6                      # every inner solve capped: the counts are all kmax
        info = s.solve_eps("DFGM", K, kmax, 1e-30, 0.1)
        assert info["inner_counts"] == [kmax] * (K + 1)
        fixed = s.solve("DFGM", K, kmax)
        assert info["matrix_passes"] == fixed["matrix_passes"], (rho, info["matrix_passes"], fixed["matrix_passes"])
        total = info["inner_iters_total"]
        assert info["matrix_passes"] == (total + 2 * (K + 1) if rho == 0.0 else 2 * total)
        s.close()


def test_eps_mode_csr_path(torch_cuda):
    prob = qpgen.sparse_banded_eq(n=3001, p=1201, seed=4)
    Qd, Gd = prob.Q.toarray(), prob.G.toarray()
    L_in, L_d, _ = O.lipschitz_constants(Qd, Gd, 5.0, 0.5)
    from paper_1504_05708_b200 import Solver
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=5.0)
    s.set_constants(L_in, L_d)
    info = s.solve_eps("DFGM", 5, 200, 1e-6, 0.5)
    xl, xa, lam = s.result()
    s.close()
    assert info["path"] == 5
    _check(prob, 5.0, "DFGM", 5, 200, 1e-6, 0.5, L_in, L_d, info, xl, xa, lam)


def test_eps_mode_rejects_bad_arguments(torch_cuda):
    from paper_1504_05708_b200 import Solver, DuquadError
    prob = qpgen.dense_ineq(50, 25, seed=0)
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0)
    s.set_constants(100.0, 1.0)
    for eps_in, sig in [(0.0, 0.1), (1e-6, 0.0), (float("nan"), 0.1)]:
        with pytest.raises(DuquadError):
            s.solve_eps("DFGM", 2, 10, eps_in, sig)
    s.close()


@pytest.mark.parametrize("P,n,p", [(2, 301, 97), (3, 4100, 1500)])
def test_eps_mode_row_sharded_emulated(torch_cuda, P, n, p):
    """Row-sharded eps_in mode (emulated ranks on one GPU): the stop test's sum is all-reduced over
    the ranks, every rank takes the same decision; two-pass (n = 301) and the row-sharded byte floor
    (n = 4100) -- the oracle replays the counts and every decision is checked."""
    from paper_1504_05708_b200 import Solver, solve_emulated_eps
    import torch
    prob = qpgen.dense_ineq(n, p, seed=3, shift=0.1)
    prob.G *= 0.05
    prob.g *= 0.05
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    eps_in, sigma_L, K, kmax = 1e-4, 0.1, 3, 120
    st = torch.cuda.Stream()
    ss = [Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0, world_size=P, rank=r,
                 emulate_ranks=True, stream=st.cuda_stream, small_path=False) for r in range(P)]
    for s in ss:
        s.set_constants(L_in, L_d)
    info = solve_emulated_eps(ss, "DFGM", K, kmax, eps_in, sigma_L)
    parts = [s.result() for s in ss]
    for s in ss:
        s.close()
    xl, xa, lam = (np.concatenate([pt[i] for pt in parts]) for i in range(3))
    info["inner_iters_total"] = sum(info["inner_counts"])
    _check(prob, 1.0, "DFGM", K, kmax, eps_in, sigma_L, L_in, L_d, info, xl, xa, lam)


def test_eps_mode_batched_per_qp_decisions(torch_cuda):
    """Batched eps_in mode: every QP of the batch stops on its own gradient-map test; the oracle
    replays each QP's counts (iterates to 1e-9) and checks each of its stop decisions."""
    from types import SimpleNamespace
    from paper_1504_05708_b200 import Solver
    B = 9
    prob = qpgen.mpc_batch(B, seed=5, N=4)                # n = 16, p = 96
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    eps_in, sigma_L, K, kmax = 1e-7, 0.1, 4, 400
    s = Solver(prob.Q, prob.q.T.copy(), prob.G, prob.g.T.copy(), prob.lb, prob.ub, prob.cone, rho=1.0)
    s.set_constants(L_in, L_d)
    info = s.solve_eps("DFGM", K, kmax, eps_in, sigma_L)
    xl, xa, lam = s.result()
    s.close()
    assert info["path"] == 4 and len(info["inner_counts"]) == B
    assert len({tuple(c) for c in info["inner_counts"]}) > 1      # the QPs stop at different steps
    for b in range(B):
        qb = SimpleNamespace(Q=prob.Q, q=prob.q[:, b], G=prob.G, g=prob.g[:, b], lb=prob.lb, ub=prob.ub,
                             cone=prob.cone)
        ib = dict(inner_counts=info["inner_counts"][b], converged=info["converged"][b],
                  inner_iters_total=sum(info["inner_counts"][b]),
                  capped=not all(info["converged"][b]))
        _check(qb, 1.0, "DFGM", K, kmax, eps_in, sigma_L, L_in, L_d, ib, xl[b], xa[b], lam[b])


@pytest.mark.parametrize("kmax", [199, 201])
def test_eps_mode_ping_pong_paths_odd_cap(torch_cuda, kmax):
    """rho = 0 (K3) with an odd inner cap: the converged solves end in either y replica, and the
    next DFOM step must read the one holding u_bar^j (the finish kernel's target)."""
    prob = qpgen.dense_ineq(600, 300, seed=2, shift=0.1)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 0.0, 0.1)
    info, xl, xa, lam = _run(prob, 0.0, "DFGM", 6, kmax, 1e-7, 0.1, L_in, L_d, small_path=False)
    assert info["path"] == 2
    _check(prob, 0.0, "DFGM", 6, kmax, 1e-7, 0.1, L_in, L_d, info, xl, xa, lam)
