"""GPU-vs-oracle parity through the C ABI (-m gpu).

Bar (BASELINE.json north_star): ||x_gpu - x_orc||_inf / (1 + ||x_orc||_inf) <= 1e-9 in fp64,
after identical fixed iteration counts with identical injected L_in, L_d (SURVEY.md §8(c)
parity protocol: short prefixes, per-outer traces, and configured counts).
"""
import numpy as np
import pytest

import qpgen
from oracle import dfom as O

pytestmark = pytest.mark.gpu

TOL = 1e-9


def relerr(got, want):
    got = np.asarray(got, dtype=float)
    want = np.asarray(want, dtype=float)
    if want.size == 0:
        return 0.0
    return float(np.max(np.abs(got - want)) / (1.0 + np.max(np.abs(want))))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _to_dev(torch, prob):
    return {k: torch.from_numpy(np.ascontiguousarray(getattr(prob, k))).to("cuda")
            for k in ("Q", "q", "G", "g", "lb", "ub", "cone")}


def run_gpu(torch, prob, rho, alg, outer, inner, L_in, L_d, trace=False, on_device=True, **opts):
    from paper_1504_05708_b200 import Solver
    if on_device:
        t = _to_dev(torch, prob)
        args = [t[k] for k in ("Q", "q", "G", "g", "lb", "ub", "cone")]
    else:
        args = [getattr(prob, k) for k in ("Q", "q", "G", "g", "lb", "ub", "cone")]
    s = Solver(*args, rho=rho, **opts)
    s.set_constants(L_in, L_d)
    tl = tu = None
    if trace:
        tl = torch.zeros((outer, max(prob.p, 1)), dtype=torch.float64, device="cuda")
        tu = torch.zeros((outer, prob.n), dtype=torch.float64, device="cuda")
        s.set_trace(tl, tu, outer)
    info = s.solve(alg, outer, inner)
    xl, xa, lam = s.result()
    out = dict(x_last=xl, x_avg=xa, lam=lam, info=info, solver=s)
    if trace:
        out["trace_lam"] = tl.cpu().numpy()[:, :prob.p]
        out["trace_u"] = tu.cpu().numpy()
    return out


def run_oracle(prob, rho, alg, outer, inner, L_in, L_d, **kw):
    return O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, alg, outer, inner,
                  L_in, L_d, **kw)


def assert_parity(g, r, trace=False):
    assert relerr(g["x_last"], r.x_last) <= TOL, relerr(g["x_last"], r.x_last)
    assert relerr(g["x_avg"], r.x_avg) <= TOL, relerr(g["x_avg"], r.x_avg)
    assert relerr(g["lam"], r.lam) <= TOL, relerr(g["lam"], r.lam)
    if trace:
        for j, (lt, ut) in enumerate(zip(r.trace_lam, r.trace_u)):
            assert relerr(g["trace_lam"][j], lt) <= TOL, ("lambda trace", j)
            assert relerr(g["trace_u"][j], ut) <= TOL, ("u trace", j)


# ------------------------------------------------------------- config 0
@pytest.fixture(scope="module")
def c0():
    return qpgen.dense_ineq(50, 25, seed=0)


def test_config0_configured_counts(torch_cuda, c0):
    """BASELINE.json configs[0]: DFGM rho = 1, 200 x 50."""
    L_in, L_d, _ = O.lipschitz_constants(c0.Q, c0.G, 1.0, 0.1)
    g = run_gpu(torch_cuda, c0, 1.0, "DFGM", 200, 50, L_in, L_d)
    r = run_oracle(c0, 1.0, O.DFGM, 200, 50, L_in, L_d)
    assert_parity(g, r)
    assert g["info"]["inner_iters_total"] == 201 * 50


@pytest.mark.parametrize("outer,inner", [(1, 1), (1, 5), (3, 5), (10, 10)])
@pytest.mark.parametrize("rho", [0.0, 1.0])
@pytest.mark.parametrize("alg", ["DGM", "DFGM"])
@pytest.mark.parametrize("project_dual", [True, False])
def test_config0_prefixes_with_trace(torch_cuda, c0, outer, inner, rho, alg, project_dual):
    """SURVEY.md §8(c) parity protocol (i): short prefixes expose convention bugs that the
    configured counts hide (dual step scale, last iterate, inner rule, K_d projection)."""
    L_in, L_d, _ = O.lipschitz_constants(c0.Q, c0.G, rho, 0.1)
    g = run_gpu(torch_cuda, c0, rho, alg, outer, inner, L_in, L_d, trace=True, project_dual=project_dual)
    r = run_oracle(c0, rho, alg, outer, inner, L_in, L_d, keep_trace=True, project_dual=project_dual)
    assert_parity(g, r, trace=True)


# ------------------------------------------------------------- config 1
@pytest.fixture(scope="module")
def c1():
    return qpgen.dense_ineq(2000, 1000, seed=0)


@pytest.fixture(scope="module")
def c1_consts(c1):
    return {rho: O.lipschitz_constants(c1.Q, c1.G, rho, 0.1) for rho in (0.0, 1.0, 10.0)}


@pytest.mark.parametrize("rho", [0.0, 1.0, 10.0])
@pytest.mark.parametrize("alg", ["DGM", "DFGM"])
def test_config1_prefix(torch_cuda, c1, c1_consts, rho, alg):
    """BASELINE.json configs[1] (n = 2000, p = 1000), rho in {0, 1, 10}, both algorithms,
    per-outer trace of (lambda^j, u_bar^j)."""
    L_in, L_d, _ = c1_consts[rho]
    g = run_gpu(torch_cuda, c1, rho, alg, 6, 8, L_in, L_d, trace=True)
    r = run_oracle(c1, rho, alg, 6, 8, L_in, L_d, keep_trace=True)
    assert_parity(g, r, trace=True)


def test_config1_longer_run(torch_cuda, c1, c1_consts):
    L_in, L_d, _ = c1_consts[1.0]
    g = run_gpu(torch_cuda, c1, 1.0, "DFGM", 40, 25, L_in, L_d)
    r = run_oracle(c1, 1.0, O.DFGM, 40, 25, L_in, L_d)
    assert_parity(g, r)


# ------------------------------------------------------------- edge cases
@pytest.mark.parametrize("n,p,kind", [(37, 13, "mixed"), (1, 1, "ineq"), (33, 0, "ineq"), (64, 64, "eq"),
                                      (97, 200, "ineq"), (5, 3, "mixed")])
def test_ragged_and_degenerate_shapes(torch_cuda, n, p, kind):
    prob = qpgen.tiny(n, p, seed=n + p, kind=kind)
    rho = 1.0
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, rho, 0.05)
    if p == 0:
        L_d = 1.0      # no multipliers: the dual step is vacuous (oracle divides by L_d)
    for alg in ("DGM", "DFGM"):
        g = run_gpu(torch_cuda, prob, rho, alg, 7, 6, L_in, L_d, trace=p > 0)
        r = run_oracle(prob, rho, O.DFGM if alg == "DFGM" else O.DGM, 7, 6, L_in, L_d, keep_trace=p > 0)
        assert_parity(g, r, trace=p > 0)


def test_singular_hessian_case2(torch_cuda):
    """Case 2: Q PSD with rank < n needs rho > 0."""
    prob = qpgen.tiny(40, 20, seed=3, kind="mixed", psd_rank=10)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 2.0, 0.0)
    g = run_gpu(torch_cuda, prob, 2.0, "DFGM", 12, 9, L_in, L_d, trace=True)
    r = run_oracle(prob, 2.0, O.DFGM, 12, 9, L_in, L_d, keep_trace=True)
    assert_parity(g, r, trace=True)


def test_infinite_box_bounds(torch_cuda):
    prob = qpgen.tiny(30, 10, seed=4, kind="eq")
    prob.lb[::3] = -np.inf
    prob.ub[1::3] = np.inf
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    g = run_gpu(torch_cuda, prob, 1.0, "DFGM", 9, 7, L_in, L_d)
    r = run_oracle(prob, 1.0, O.DFGM, 9, 7, L_in, L_d)
    assert_parity(g, r)


@pytest.mark.parametrize("rule", ["GM", "FGM_SIGMA"])
def test_inner_rules(torch_cuda, c0, rule):
    L_in, L_d, _ = O.lipschitz_constants(c0.Q, c0.G, 1.0, 0.1)
    sigma = 0.1 if rule == "FGM_SIGMA" else 0.0
    g = run_gpu(torch_cuda, c0, 1.0, "DFGM", 8, 6, L_in, L_d, inner_rule=rule, sigma=sigma)
    r = run_oracle(c0, 1.0, O.DFGM, 8, 6, L_in, L_d,
                   inner_rule=O.INNER_GM if rule == "GM" else O.INNER_FGM_SIGMA, sigma=sigma)
    assert_parity(g, r)


def test_dual_step_scale_option(torch_cuda, c0):
    L_in, L_d, _ = O.lipschitz_constants(c0.Q, c0.G, 1.0, 0.1)
    g = run_gpu(torch_cuda, c0, 1.0, "DGM", 5, 5, L_in, L_d, dual_step_scale=1.0)
    r = run_oracle(c0, 1.0, O.DGM, 5, 5, L_in, L_d, dual_step_scale=1.0)
    assert_parity(g, r)


def test_host_and_device_inputs_agree_bitwise(torch_cuda, c0):
    L_in, L_d, _ = O.lipschitz_constants(c0.Q, c0.G, 1.0, 0.1)
    a = run_gpu(torch_cuda, c0, 1.0, "DFGM", 10, 10, L_in, L_d, on_device=True)
    b = run_gpu(torch_cuda, c0, 1.0, "DFGM", 10, 10, L_in, L_d, on_device=False)
    c = run_gpu(torch_cuda, c0, 1.0, "DFGM", 10, 10, L_in, L_d, use_graphs=False)
    for k in ("x_last", "x_avg", "lam"):
        assert np.array_equal(a[k], b[k]) and np.array_equal(a[k], c[k]), k


def test_repeat_solve_is_deterministic(torch_cuda, c1, c1_consts):
    L_in, L_d, _ = c1_consts[1.0]
    g = run_gpu(torch_cuda, c1, 1.0, "DFGM", 5, 5, L_in, L_d)
    s = g["solver"]
    s.solve("DFGM", 5, 5)
    xl, xa, lam = s.result()
    assert np.array_equal(xl, g["x_last"]) and np.array_equal(lam, g["lam"])


# ------------------------------------------------------------- constants / residuals / errors
def test_lipschitz_matches_eigvalsh(torch_cuda, c1):
    from paper_1504_05708_b200 import Solver
    for rho, l_mode in ((1.0, 0), (10.0, 0), (1.0, 1), (0.0, 0)):
        s = Solver(c1.Q, c1.q, c1.G, c1.g, c1.lb, c1.ub, c1.cone, rho=rho, lambda_min_lb=0.1, l_mode=l_mode)
        L_in, L_d, nG2 = s.lipschitz(iters=150, safety=0.0)
        rL, rd, rn = O.lipschitz_constants(c1.Q, c1.G, rho, 0.1, l_mode=l_mode)
        assert abs(nG2 - rn) <= 1e-9 * rn
        assert abs(L_in - rL) <= 1e-9 * rL, (rho, l_mode, L_in, rL)
        assert abs(L_d - rd) <= 1e-9 * rd
        s.close()


def test_residuals_match_oracle(torch_cuda, c0):
    rho = 1.0
    L_in, L_d, _ = O.lipschitz_constants(c0.Q, c0.G, rho, 0.1)
    g = run_gpu(torch_cuda, c0, rho, "DFGM", 30, 20, L_in, L_d)
    r = run_oracle(c0, rho, O.DFGM, 30, 20, L_in, L_d)
    for which, x in (("last", r.x_last), ("avg", r.x_avg)):
        F, dist, lag = g["solver"].residuals(which)
        assert abs(F - O.objective(c0.Q, c0.q, x)) <= 1e-9 * (1 + abs(F))
        assert abs(dist - O.dist_K(c0.G @ x + c0.g, c0.cone)) <= 1e-9 * (1 + dist)
        ref_lag = O.aug_lagrangian(c0.Q, c0.q, c0.G, c0.g, c0.cone, rho, x, r.lam)
        assert abs(lag - ref_lag) <= 1e-9 * (1 + abs(ref_lag))


def test_solve_before_constants_is_an_error(torch_cuda, c0):
    from paper_1504_05708_b200 import Solver, DuquadError
    s = Solver(c0.Q, c0.q, c0.G, c0.g, c0.lb, c0.ub, c0.cone, rho=1.0)
    with pytest.raises(DuquadError) as e:
        s.solve("DFGM", 1, 1)
    assert e.value.status == 7
    with pytest.raises(DuquadError):
        s.set_constants(-1.0, 1.0)


def test_nonfinite_iterates_are_reported(torch_cuda, c0):
    from paper_1504_05708_b200 import Solver, DuquadError
    prob = qpgen.tiny(20, 5, seed=1)
    prob.lb[:] = -np.inf
    prob.ub[:] = np.inf
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0)
    s.set_constants(1e-12, 1e-12)          # far too small L: the iteration blows up
    with pytest.raises(DuquadError) as e:
        s.solve("DFGM", 50, 50)
    assert e.value.status == 5


def test_device_input_validation(torch_cuda, c0):
    from paper_1504_05708_b200 import Solver, DuquadError
    t = _to_dev(torch_cuda, c0)
    t["Q"][3, 4] = float("nan")
    with pytest.raises(DuquadError) as e:
        Solver(t["Q"], t["q"], t["G"], t["g"], t["lb"], t["ub"], t["cone"], rho=1.0)
    assert e.value.status == 1


def test_host_input_validation_on_device(torch_cuda, c0):
    """A single rank's host Q and G are checked for non-finite values on the device after their
    upload (no host scan): a NaN / inf in Q or G is still rejected with EINVAL, and an emulated
    2-rank setup (host scan) rejects it alike."""
    from paper_1504_05708_b200 import Solver, DuquadError
    for name, (i, j), v in (("Q", (3, 4), float("nan")), ("G", (7, 11), float("inf")),
                            ("G", (c0.G.shape[0] - 1, c0.G.shape[1] - 1), float("nan"))):
        arrs = {k: getattr(c0, k).copy() for k in ("Q", "G")}
        arrs[name][i, j] = v
        for kw in ({}, dict(world_size=2, rank=1, emulate_ranks=True)):
            with pytest.raises(DuquadError, match="non-finite") as e:
                Solver(arrs["Q"], c0.q, arrs["G"], c0.g, c0.lb, c0.ub, c0.cone, rho=1.0, **kw)
            assert e.value.status == 1


# ------------------------------------------------------------- config 2 at full size
@pytest.mark.slow
def test_config2_full_size_prefix(torch_cuda):
    """BASELINE.json configs[2] at full size (n = 16384, p = 8192) in the bench's launch
    configuration: a 2 x 2 prefix (6 inner steps incl. the last-iterate solve) against the
    oracle on the host, plus the full-length DFGM solve's lambda in K_d."""
    from paper_1504_05708_b200 import Solver
    d = qpgen.dense_ineq_torch(16384, 8192, seed=0, shift=0.05)
    s = Solver(d["Q"], d["q"], d["G"], d["g"], d["lb"], d["ub"], d["cone"], rho=1.0, lambda_min_lb=0.05)
    L_in, L_d, _ = s.lipschitz(iters=60, safety=1e-3)
    s.solve("DFGM", 2, 2)
    xl, xa, lam = s.result()
    h = {k: v.cpu().numpy() for k, v in d.items()}
    r = O.dfom(h["Q"], h["q"], h["G"], h["g"], h["lb"], h["ub"], h["cone"], 1.0, O.DFGM, 2, 2, L_in, L_d)
    assert relerr(xl, r.x_last) <= TOL and relerr(xa, r.x_avg) <= TOL and relerr(lam, r.lam) <= TOL
    s.close()


@pytest.mark.parametrize("n,p,kind", [(50, 25, "ineq"), (37, 13, "mixed"), (33, 0, "ineq"), (90, 45, "eq")])
def test_small_whole_solve_kernel_matches_the_stream_path(torch_cuda, n, p, kind):
    """K4 (one CTA runs the whole solve from shared memory, one thread per row) vs the two-kernel
    streaming path: the same epilogues, a different summation order -> agreement to 1e-12, and both
    at parity with the oracle."""
    prob = qpgen.tiny(n, p, seed=n, kind=kind)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.05)
    L_d = L_d if p else 1.0
    a = run_gpu(torch_cuda, prob, 1.0, "DFGM", 9, 7, L_in, L_d, trace=p > 0, small_path=True)
    b = run_gpu(torch_cuda, prob, 1.0, "DFGM", 9, 7, L_in, L_d, trace=p > 0, small_path=False, persist_path=False)
    assert a["info"]["kernel_launches"] == 2 and b["info"]["kernel_launches"] > 2
    for k in ("x_last", "x_avg", "lam") + (("trace_lam", "trace_u") if p else ()):
        assert relerr(a[k], b[k]) <= 1e-12, k
    r = run_oracle(prob, 1.0, O.DFGM, 9, 7, L_in, L_d)
    assert_parity(a, r)


@pytest.mark.parametrize("alg", ["DGM", "DFGM"])
@pytest.mark.parametrize("K,Kin", [(1, 1), (3, 4), (6, 5)])
def test_rho0_q_only_inner_step(torch_cuda, c1, c1_consts, alg, K, Kin):
    """Row a1' (rho = 0): K3 streams Q only per inner step, c = q + G'mu per outer iteration
    (P:1268-1270); parity with the oracle incl. per-outer traces, odd and even K_in (ping-pong)."""
    L_in, L_d, _ = c1_consts[0.0]
    g = run_gpu(torch_cuda, c1, 0.0, alg, K, Kin, L_in, L_d, trace=True)
    assert g["info"]["kernel_launches"] == 1 + (K + 1) * (Kin + 3)
    r = run_oracle(c1, 0.0, alg, K, Kin, L_in, L_d, keep_trace=True)
    assert_parity(g, r, trace=True)
    h = run_gpu(torch_cuda, c1, 0.0, alg, K, Kin, L_in, L_d, rho0_path=False)
    assert relerr(g["x_last"], h["x_last"]) <= 1e-13 and relerr(g["lam"], h["lam"]) <= 1e-13


def test_asymmetric_q_is_rejected(torch_cuda):
    """Q must be symmetric; the library checks dense Q at setup (single GPU)."""
    from paper_1504_05708_b200 import Solver, DuquadError
    prob = qpgen.tiny(40, 10, seed=9)
    Q = prob.Q.copy()
    Q[3, 17] += 1e-6
    with pytest.raises(DuquadError, match="symmetric"):
        Solver(Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0)
    Q = prob.Q.copy()
    Q[3, 17] *= 1.0 + 1e-15    # rounding-level asymmetry is accepted
    Solver(Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0).close()


def test_asymmetric_q_is_rejected_on_every_rank_count_and_format(torch_cuda):
    """The symmetry check is not a single-GPU special case: a row-sharded rank (which holds only its
    rows) checks the caller's full Q -- host or device input, both byte-floor and two-pass sizes --
    and the CSR path compares Q with its transpose."""
    import scipy.sparse as sp
    from paper_1504_05708_b200 import Solver, DuquadError
    for n, p in ((40, 10), (4096, 256)):
        prob = qpgen.tiny(n, p, seed=9)
        Q = prob.Q.copy()
        Q[30, 3] += 1e-6           # below the diagonal: rank 1's rows
        for dev in (False, True):
            Qa = torch_cuda.from_numpy(Q).cuda() if dev else Q
            args = [torch_cuda.from_numpy(a).cuda() if dev else a for a in (prob.q, prob.G, prob.g, prob.lb, prob.ub,
                                                                           prob.cone)]
            for r in range(2):
                with pytest.raises(DuquadError, match="symmetric"):
                    Solver(Qa, *args, rho=1.0, world_size=2, rank=r, emulate_ranks=True)
    prob = qpgen.sparse_banded_eq(n=300, p=100, seed=3)
    Q = prob.Q.tolil()
    Q[5, 7] = Q[5, 7] + 1e-6
    with pytest.raises(DuquadError, match="symmetric"):
        Solver(sp.csr_matrix(Q), prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=5.0)
    Q = prob.Q.tolil()
    Q[5, 150] = 0.3            # an entry without its mirror: the pattern is not symmetric
    with pytest.raises(DuquadError, match="symmetric"):
        Solver(sp.csr_matrix(Q), prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=5.0)
    Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=5.0).close()   # symmetric: accepted


@pytest.mark.parametrize("n,p,kind,rho,alg", [(2000, 1000, "ineq", 1.0, "DFGM"), (2000, 1000, "ineq", 10.0, "DGM"),
                                               (777, 301, "mixed", 2.0, "DFGM"), (130, 0, "ineq", 1.0, "DFGM")])
def test_persistent_solve_is_bitwise_the_multi_launch_path(torch_cuda, n, p, kind, rho, alg):
    """k_persist (one cooperative launch per solve, grid barriers between the passes) vs one launch
    per pass: the same row sums and epilogues -> bit-identical; and parity with the oracle."""
    prob = qpgen.dense_ineq(n, p, seed=0) if kind == "ineq" and n == 2000 else qpgen.tiny(n, p, seed=n, kind=kind)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, rho, 0.1)
    L_d = L_d if p else 1.0
    a = run_gpu(torch_cuda, prob, rho, alg, 7, 9, L_in, L_d, small_path=False, persist_path=True)
    b = run_gpu(torch_cuda, prob, rho, alg, 7, 9, L_in, L_d, small_path=False, persist_path=False)
    assert a["info"]["path"] == 7 and b["info"]["path"] == 0
    for k in ("x_last", "x_avg", "lam"):
        assert np.array_equal(a[k], b[k]), k
    r = run_oracle(prob, rho, O.DFGM if alg == "DFGM" else O.DGM, 7, 9, L_in, L_d)
    assert_parity(a, r)


@pytest.mark.parametrize("kind", ["two_pass", "byte_floor", "rho0", "batched"])
def test_pdl_launch_does_not_change_results(torch_cuda, kind):
    """Programmatic dependent launch (options.pdl) only overlaps a kernel's launch and matrix
    prefetch with its predecessor; every read of an iterate happens after the dependency wait, so
    the iterates are bitwise those of plain launches (graph-captured, several outer iterations)."""
    from paper_1504_05708_b200 import Solver
    if kind == "batched":
        prob = qpgen.mpc_batch(300, seed=3, N=12)
        args = (prob.Q, prob.q.T.copy(), prob.G, prob.g.T.copy(), prob.lb, prob.ub, prob.cone)
        kw, rho = {}, 1.0
    else:
        n, p = (4096, 700) if kind == "byte_floor" else (900, 400)
        prob = qpgen.tiny(n, p, seed=17, kind="mixed", shift=0.2)
        args = (prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone)
        kw = dict(small_path=False, fused_path=kind == "byte_floor")
        rho = 0.0 if kind == "rho0" else 1.0
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, rho, 0.2 if kind != "batched" else 0.1)
    outs = []
    for pdl in (True, False):
        s = Solver(*args, rho=rho, pdl=pdl, **kw)
        s.set_constants(L_in, L_d)
        info = s.solve("DFGM", 5, 6)
        outs.append(s.result())
        s.close()
    want = {"two_pass": 0, "byte_floor": 1, "rho0": 2, "batched": 4}[kind]
    assert info["path"] == want, info["path"]
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
