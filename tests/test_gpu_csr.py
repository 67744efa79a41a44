"""CSR path (BASELINE.json configs[4]) vs the oracle (-m gpu)."""
import numpy as np
import pytest
import scipy.sparse as sp

import qpgen
from oracle import dfom as O

pytestmark = pytest.mark.gpu
TOL = 1e-9


def relerr(got, want):
    got, want = np.asarray(got, float), np.asarray(want, float)
    if want.size == 0:
        return 0.0
    return float(np.max(np.abs(got - want)) / (1.0 + np.max(np.abs(want))))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _consts_dense(prob, rho, lmin):
    return O.lipschitz_constants(prob.Q.toarray(), prob.G.toarray(), rho, lmin)


def _gpu(prob, rho, alg, K, Kin, L_in, L_d, trace=False, torch=None, **kw):
    from paper_1504_05708_b200 import Solver
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=rho, **kw)
    s.set_constants(L_in, L_d)
    out = {}
    if trace:
        tl = torch.zeros((K, max(prob.p, 1)), dtype=torch.float64, device="cuda")
        tu = torch.zeros((K, prob.n), dtype=torch.float64, device="cuda")
        s.set_trace(tl, tu, K)
    s.solve(alg, K, Kin)
    out["x_last"], out["x_avg"], out["lam"] = s.result()
    if trace:
        out["trace_lam"] = tl.cpu().numpy()[:, :prob.p]
        out["trace_u"] = tu.cpu().numpy()
    out["solver"] = s
    return out


def _check(g, r, trace=False):
    assert relerr(g["x_last"], r.x_last) <= TOL
    assert relerr(g["x_avg"], r.x_avg) <= TOL
    assert relerr(g["lam"], r.lam) <= TOL
    if trace:
        for j in range(len(r.trace_lam)):
            assert relerr(g["trace_lam"][j], r.trace_lam[j]) <= TOL, j
            assert relerr(g["trace_u"][j], r.trace_u[j]) <= TOL, j


@pytest.mark.parametrize("alg", ["DGM", "DFGM"])
@pytest.mark.parametrize("K,Kin", [(1, 1), (3, 5), (12, 10)])
def test_banded_small_parity_with_trace(torch_cuda, alg, K, Kin):
    prob = qpgen.sparse_banded_eq(n=300, p=100, seed=3)
    L_in, L_d, _ = _consts_dense(prob, 5.0, 0.5)
    g = _gpu(prob, 5.0, alg, K, Kin, L_in, L_d, trace=True, torch=torch_cuda)
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 5.0, alg, K, Kin, L_in, L_d,
               keep_trace=True)
    _check(g, r, trace=True)


@pytest.mark.parametrize("kind,rho", [("ineq", 1.0), ("mixed", 0.0), ("eq", 2.0)])
def test_random_sparse_cones(torch_cuda, kind, rho):
    """Sparse versions of the tiny families (inequality / mixed / equality, rho = 0 too)."""
    d = qpgen.tiny(150, 60, seed=7, kind=kind)
    rng = np.random.default_rng(1)
    mask = rng.random(d.G.shape) < 0.1
    G = sp.csr_matrix(np.where(mask, d.G, 0.0))
    g = -(G @ d.meta["x0"]) - np.where(d.cone == qpgen.NONPOS, 0.3, 0.0)
    Q = sp.csr_matrix(np.where(np.abs(d.Q) > 0.05, d.Q, 0.0) + 0.5 * np.eye(150))
    prob = qpgen.SparseQP(Q, d.q, G, g, d.lb, d.ub, d.cone)
    lmin = float(np.linalg.eigvalsh(Q.toarray())[0])
    assert lmin > 0
    L_in, L_d, _ = O.lipschitz_constants(Q.toarray(), G.toarray(), rho, lmin)
    g_ = _gpu(prob, rho, "DFGM", 9, 8, L_in, L_d)
    r = O.dfom(Q, d.q, G, g, d.lb, d.ub, d.cone, rho, O.DFGM, 9, 8, L_in, L_d)
    _check(g_, r)


def test_csr_matches_dense_path(torch_cuda):
    """The same QP through the dense and the CSR kernels (different summation order only)."""
    from paper_1504_05708_b200 import Solver
    prob = qpgen.sparse_banded_eq(n=500, p=200, seed=5)
    L_in, L_d, _ = _consts_dense(prob, 5.0, 0.5)
    a = _gpu(prob, 5.0, "DFGM", 20, 10, L_in, L_d)
    s = Solver(prob.Q.toarray(), prob.q, prob.G.toarray(), prob.g, prob.lb, prob.ub, prob.cone, rho=5.0)
    s.set_constants(L_in, L_d)
    s.solve("DFGM", 20, 10)
    xl, xa, lam = s.result()
    assert relerr(a["x_last"], xl) <= 1e-12 and relerr(a["lam"], lam) <= 1e-12


def test_device_csr_inputs_and_lipschitz(torch_cuda):
    from paper_1504_05708_b200 import Solver
    torch = torch_cuda
    prob = qpgen.sparse_banded_eq(n=400, p=150, seed=9)
    Q, G = prob.Q, prob.G
    dv = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype=dt)
    s = Solver.csr(400, 150, dv(Q.indptr, torch.int32), dv(Q.indices, torch.int32), dv(Q.data, torch.float64),
                   dv(G.indptr, torch.int32), dv(G.indices, torch.int32), dv(G.data, torch.float64),
                   dv(prob.q, torch.float64), dv(prob.g, torch.float64), dv(prob.lb, torch.float64),
                   dv(prob.ub, torch.float64), dv(prob.cone, torch.uint8), rho=5.0, lambda_min_lb=0.5)
    L_in, L_d, nG2 = s.lipschitz(iters=120, safety=0.0)
    rL, rd, rn = _consts_dense(prob, 5.0, 0.5)
    assert abs(L_in - rL) <= 1e-9 * rL and abs(nG2 - rn) <= 1e-9 * rn and abs(L_d - rd) <= 1e-9 * rd
    s.set_constants(rL, rd)
    s.solve("DGM", 6, 7)
    xl, xa, lam = s.result()
    r = O.dfom(Q, prob.q, G, prob.g, prob.lb, prob.ub, prob.cone, 5.0, O.DGM, 6, 7, rL, rd)
    assert relerr(xl, r.x_last) <= TOL and relerr(lam, r.lam) <= TOL


def test_invalid_csr_is_rejected(torch_cuda):
    from paper_1504_05708_b200 import Solver, DuquadError
    prob = qpgen.sparse_banded_eq(n=50, p=10, seed=1)
    G = prob.G.copy()
    G.indices[3] = 50          # column out of range
    with pytest.raises(DuquadError) as e:
        Solver(prob.Q, prob.q, G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0)
    assert e.value.status == 1


@pytest.fixture(scope="module")
def c4():
    return qpgen.sparse_banded_eq()      # BASELINE.json configs[4] at full size


def test_config4_full_size_prefix(torch_cuda, c4):
    """configs[4] at full size (n = 1e6, p = 5e5, 15M + 4M nnz) in the bench launch configuration:
    DFGM and DGM rho = 5 prefixes against the SciPy-CSR oracle, with per-outer trace."""
    from paper_1504_05708_b200 import Solver
    s = Solver(c4.Q, c4.q, c4.G, c4.g, c4.lb, c4.ub, c4.cone, rho=5.0, lambda_min_lb=0.5)
    L_in, L_d, nG2 = s.lipschitz(iters=40, safety=1e-3)
    assert 5.0 * nG2 <= L_in <= (3.0 + 5.0 * nG2) * 1.01       # lambda_max(Q) <= 3 (Gershgorin)
    s.close()
    for alg in ("DFGM", "DGM"):
        g = _gpu(c4, 5.0, alg, 4, 6, L_in, L_d, trace=True, torch=torch_cuda)
        r = O.dfom(c4.Q, c4.q, c4.G, c4.g, c4.lb, c4.ub, c4.cone, 5.0, alg, 4, 6, L_in, L_d, keep_trace=True)
        _check(g, r, trace=True)


def test_csr_empty_rows(torch_cuda):
    """CSR rows without nonzeros (in G and in the stacked [Q;G]) next to regular ones."""
    import scipy.sparse as sp
    from paper_1504_05708_b200 import Solver
    prob = qpgen.sparse_banded_eq(n=3001, p=1201, seed=7)
    G = prob.G.tolil()
    for r in (0, 5, 600, 1200):
        G.rows[r] = []
        G.data[r] = []
    G = G.tocsr()
    g = prob.g.copy()
    g[[0, 5, 600, 1200]] = 0.0
    Gd = G.toarray()
    L_in, L_d, _ = O.lipschitz_constants(prob.Q.toarray(), Gd, 5.0, 0.5)
    s = Solver(prob.Q, prob.q, G, g, prob.lb, prob.ub, prob.cone, rho=5.0)
    s.set_constants(L_in, L_d)
    assert s.solve("DFGM", 3, 4)["path"] == 5
    got = s.result()
    s.close()
    r = O.dfom(prob.Q, prob.q, G, g, prob.lb, prob.ub, prob.cone, 5.0, "DFGM", 3, 4, L_in, L_d)
    for a, b in zip(got, (r.x_last, r.x_avg, r.lam)):
        assert relerr(a, b) <= 1e-9, relerr(a, b)


# ------------------------------------------------------------------ lane-per-row kernels (sell_path)
SELL, ROWT = 1, 2


def _skewed(n=2500, p=900, seed=11):
    """Rows of very different lengths: a banded Q plus a few denser symmetric rows, and G rows with
    1..40 nonzeros (mean 20.5), so SELL-32 would pad too much and both passes take the
    thread-per-row CSR kernels."""
    rng = np.random.default_rng(seed)
    base = qpgen.sparse_banded_eq(n=n, p=p, seed=seed)
    Q = base.Q.tolil()
    for i in rng.choice(n, 40, replace=False):          # denser symmetric rows / columns
        cols = rng.choice(n, 12, replace=False)
        v = rng.uniform(-0.01, 0.01, 12)
        for c, x in zip(cols, v):
            if c != i:
                Q[i, c] = Q[i, c] + x
                Q[c, i] = Q[c, i] + x
    Q = sp.csr_matrix(Q)
    Q.sort_indices()
    lens = rng.integers(1, 41, p)
    rows = np.repeat(np.arange(p), lens)
    cols = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens])
    G = sp.csr_matrix((rng.standard_normal(len(cols)), (rows, cols)), shape=(p, n))
    G.sort_indices()
    x0 = rng.uniform(-0.5, 0.5, n)
    cone = np.where(np.arange(p) % 3 == 0, qpgen.NONPOS, qpgen.ZERO).astype(np.uint8)
    g = -(G @ x0) - np.where(cone == qpgen.NONPOS, 0.2, 0.0)
    return qpgen.SparseQP(Q, base.q, G, g, base.lb, base.ub, cone)


@pytest.mark.parametrize("maker,kinds", [("banded", (SELL, ROWT)), ("skewed", (ROWT, ROWT)), ("box", (SELL, ROWT))])
@pytest.mark.parametrize("alg", ["DGM", "DFGM"])
def test_lane_kernels_vs_subwarp_kernels_and_oracle(torch_cuda, maker, kinds, alg):
    """The lane-per-row kernels -- SELL-32 for the banded config-4 family's [Q;G] (rows of 11 and 8
    nonzeros), thread-per-row CSR for its G' (Poisson(4) rows) and for skewed rows -- against the
    sub-warp CSR kernels (same row sums up to summation order: 1e-12) and the oracle (1e-9), with
    the per-outer trace."""
    prob = qpgen.sparse_banded_eq(n=3001, p=1201, seed=2) if maker != "skewed" else _skewed()
    if maker == "box":   # per-coordinate bounds (the uniform-box shortcut off), some infinite
        rng = np.random.default_rng(4)
        prob.lb = -rng.uniform(0.5, 1.5, prob.lb.shape)
        prob.ub = rng.uniform(0.5, 1.5, prob.ub.shape)
        prob.lb[::7] = -np.inf
        prob.ub[3::11] = np.inf
    rho = 2.0 if maker == "skewed" else 5.0
    L_in, L_d, _ = _consts_dense(prob, rho, 0.5)
    a = _gpu(prob, rho, alg, 6, 7, L_in, L_d, trace=True, torch=torch_cuda)
    info = a["solver"].solve(alg, 6, 7)
    sk = info["sparse_kernels"]
    assert info["path"] == 5 and (sk & 3, (sk >> 4) & 3) == kinds, info
    assert bool(sk & 8) == (maker != "skewed")       # banded Q rows read as diagonals (DIA)
    assert bool(sk & 64) == (maker != "skewed")      # ... only the band's upper half stored (symmetric)
    b = _gpu(prob, rho, alg, 6, 7, L_in, L_d, sell_path=False)
    assert b["solver"].solve(alg, 6, 7)["sparse_kernels"] == 0
    for k in ("x_last", "x_avg", "lam"):
        assert relerr(a[k], b[k]) <= 1e-12, k
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, alg, 6, 7, L_in, L_d,
               keep_trace=True)
    _check(a, r, trace=True)
    a["solver"].close()
    b["solver"].close()


def test_lane_kernels_deterministic_and_serve_lipschitz_and_residuals(torch_cuda):
    """Two lane-kernel solves are bitwise identical (fixed per-row order); the MODE_LIN launches
    (Lanczos, residuals: Q-rows-only / G-rows-only sub-ranges of the stacked SELL storage) run on
    the lane kernels and match the sub-warp kernels."""
    from paper_1504_05708_b200 import Solver
    for prob, rho in ((qpgen.sparse_banded_eq(n=2000, p=700, seed=12), 5.0), (_skewed(seed=12), 2.0)):
        L_in, L_d, _ = _consts_dense(prob, rho, 0.5)
        outs, lips, res = [], [], []
        for sell in (True, True, False):
            s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=rho, lambda_min_lb=0.5,
                       sell_path=sell)
            lips.append(s.lipschitz(iters=60, safety=0.0))
            s.set_constants(L_in, L_d)
            s.solve("DFGM", 5, 6)
            outs.append(s.result())
            res.append(s.residuals("last"))
            s.close()
        for x, y in zip(outs[0], outs[1]):
            assert np.array_equal(x, y)
        for x, y in zip(outs[0], outs[2]):
            assert relerr(x, y) <= 1e-12
        assert np.allclose(lips[0], lips[2], rtol=1e-10, atol=0)
        assert np.allclose(res[0], res[2], rtol=1e-10, atol=1e-12)


def test_long_rows_keep_the_subwarp_kernels(torch_cuda):
    """Mean row length above 48 (G rows of 80 nonzeros): both passes keep the sub-warp CSR
    kernels; a G with one 400-nonzero row per 32 rows (SELL would pad > 15 %) takes thread-per-row
    CSR for [Q;G].  Both agree with the oracle."""
    from paper_1504_05708_b200 import Solver
    rng = np.random.default_rng(5)
    for n, p, lens, kind_a in ((200, 400, np.full(400, 80), 0), (1500, 64, np.where(np.arange(64) % 32 == 0, 400, 1), ROWT)):
        base = qpgen.sparse_banded_eq(n=n, p=p, seed=5)
        rows = np.repeat(np.arange(p), lens)
        cols = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens])
        G = sp.csr_matrix((rng.standard_normal(len(cols)), (rows, cols)), shape=(p, n))
        G.sort_indices()
        g = -(G @ rng.uniform(-0.5, 0.5, n))
        prob = qpgen.SparseQP(base.Q, base.q, G, g, base.lb, base.ub, base.cone)
        L_in, L_d, _ = _consts_dense(prob, 5.0, 0.5)
        s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=5.0)
        s.set_constants(L_in, L_d)
        info = s.solve("DFGM", 3, 4)
        assert info["sparse_kernels"] & 15 == kind_a, info["sparse_kernels"]
        got = s.result()
        s.close()
        r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 5.0, "DFGM", 3, 4, L_in, L_d)
        for a_, b_ in zip(got, (r.x_last, r.x_avg, r.lam)):
            assert relerr(a_, b_) <= TOL


def _perturbed_mirror(Q, i, j, rel):
    """Q with Q[i, j] (not Q[j, i]) scaled by 1 + rel: symmetric within setup's 1e-12 tolerance but
    not bitwise."""
    Q = Q.tolil(copy=True)
    Q[i, j] = Q[i, j] * (1.0 + rel)
    Q = Q.tocsr()
    Q.sort_indices()
    return Q


@pytest.mark.parametrize("half_band", [1, 5, 7])
def test_symmetric_half_band_dia(torch_cuda, monkeypatch, half_band):
    """Pass A's banded Q rows from the stored upper half of the band (symmetric DIA: Q[i, i-o] read
    as the stored Q[i-o, i]), summed in the same ascending column order: bitwise the
    full-band DIA kernels' iterates for a bitwise symmetric Q, and the oracle's to 1e-9 with the
    per-outer trace; a Q that is symmetric only to within setup's 1e-12 tolerance (one mirrored value
    1e-14 off) keeps the full band."""
    prob = qpgen.sparse_banded_eq(n=2500, p=900, seed=21, half_band=half_band)
    L_in, L_d, _ = _consts_dense(prob, 5.0, 0.5)
    a = _gpu(prob, 5.0, "DFGM", 5, 6, L_in, L_d, trace=True, torch=torch_cuda)
    assert a["solver"].solve("DFGM", 5, 6)["sparse_kernels"] & (8 | 64) == 8 | 64
    monkeypatch.setenv("DUQUAD_DIA_SYM", "0")
    b = _gpu(prob, 5.0, "DFGM", 5, 6, L_in, L_d)
    assert b["solver"].solve("DFGM", 5, 6)["sparse_kernels"] & (8 | 64) == 8
    monkeypatch.delenv("DUQUAD_DIA_SYM")
    for k in ("x_last", "x_avg", "lam"):
        assert np.array_equal(a[k], b[k]), k
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 5.0, "DFGM", 5, 6, L_in, L_d,
               keep_trace=True)
    _check(a, r, trace=True)
    a["solver"].close()
    b["solver"].close()
    # not bitwise symmetric: the full band is kept, and the oracle (which uses Q as given) agrees
    Qp = _perturbed_mirror(prob.Q, 1200, 1200 - half_band, 1e-14)
    pp = qpgen.SparseQP(Qp, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone)
    c = _gpu(pp, 5.0, "DFGM", 5, 6, L_in, L_d)
    assert c["solver"].solve("DFGM", 5, 6)["sparse_kernels"] & (8 | 64) == 8
    r = O.dfom(Qp, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 5.0, "DFGM", 5, 6, L_in, L_d)
    _check(c, r)
    c["solver"].close()


@pytest.mark.parametrize("n,P", [(3001, 3), (37, 5)])
def test_symmetric_half_band_dia_row_sharded(torch_cuda, n, P):
    """Row shards of the symmetric half band: each rank fills the halo rows before its slice from
    its own rows' lower entries (no remote data), down to slices shorter than the halo (n = 37 over
    5 ranks, half band 7): the emulated ranks' iterates equal the 1-GPU solve bit for bit and match
    the oracle."""
    from paper_1504_05708_b200 import Solver, solve_emulated
    prob = qpgen.sparse_banded_eq(n=n, p=max(n // 3, 4), seed=23, half_band=7)
    L_in, L_d, _ = _consts_dense(prob, 5.0, 0.5)
    args = [prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone]
    stream = torch_cuda.cuda.Stream().cuda_stream
    ss = [Solver(*args, rho=5.0, world_size=P, rank=r, emulate_ranks=True, stream=stream) for r in range(P)]
    for s_ in ss:
        s_.set_constants(L_in, L_d)
    solve_emulated(ss, "DFGM", 4, 5)
    parts = [s_.result() for s_ in ss]
    for s_ in ss:
        s_.close()
    got = [np.concatenate([pt[i] for pt in parts]) for i in range(3)]
    one = _gpu(prob, 5.0, "DFGM", 4, 5, L_in, L_d)
    assert one["solver"].solve("DFGM", 4, 5)["sparse_kernels"] & 64
    for g_, k in zip(got, ("x_last", "x_avg", "lam")):
        assert np.array_equal(g_, one[k]), k
    one["solver"].close()
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 5.0, "DFGM", 4, 5, L_in, L_d)
    for g_, w_ in zip(got, (r.x_last, r.x_avg, r.lam)):
        assert relerr(g_, w_) <= TOL
