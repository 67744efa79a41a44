"""Row-sharded path on ONE GPU via emulated ranks (-m gpu).

P contexts (ranks 0..P-1 of one QP, each holding only its rows of [Q;G] and G') run the solve
schedule in lock step (duquad_solve_emulated); the NCCL all-gathers of the y and w replicas are
replaced by device copies.  Every row product is independent of the sharding, so the
concatenated local results must equal the 1-GPU results BIT FOR BIT, and match the oracle.
"""
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


def relerr(got, want):
    got, want = np.asarray(got, float), np.asarray(want, float)
    return float(np.max(np.abs(got - want)) / (1.0 + np.max(np.abs(want)))) if want.size else 0.0


def _run_sharded(torch, args, P, rho, alg, K, Kin, L_in, L_d, trace=False, **kw):
    from paper_1504_05708_b200 import Solver, solve_emulated
    stream = torch.cuda.Stream().cuda_stream          # one non-default stream shared by the ranks
    ss = [Solver(*args, rho=rho, world_size=P, rank=r, emulate_ranks=True, stream=stream, **kw) for r in range(P)]
    traces = []
    for s in ss:
        s.set_constants(L_in, L_d)
        if trace:
            nl = s.n_range[1] - s.n_range[0]
            pl = s.p_range[1] - s.p_range[0]
            tl = torch.zeros((K, max(pl, 1)), dtype=torch.float64, device="cuda")
            tu = torch.zeros((K, max(nl, 1)), dtype=torch.float64, device="cuda")
            s.set_trace(tl, tu, K)
            traces.append((tl, tu, pl, nl))
    solve_emulated(ss, alg, K, Kin)
    parts = [s.result() for s in ss]
    out = {k: np.concatenate([pt[i] for pt in parts]) for i, k in enumerate(("x_last", "x_avg", "lam"))}
    if trace:
        out["trace_lam"] = np.concatenate([tl.cpu().numpy()[:, :pl] for tl, tu, pl, nl in traces], axis=1)
        out["trace_u"] = np.concatenate([tu.cpu().numpy()[:, :nl] for tl, tu, pl, nl in traces], axis=1)
    for s in ss:
        s.close()
    return out


def _run_single(torch, args, rho, alg, K, Kin, L_in, L_d, trace=False, **kw):
    from paper_1504_05708_b200 import Solver
    s = Solver(*args, rho=rho, small_path=False, fused_path=False, **kw)
    s.set_constants(L_in, L_d)
    if trace:
        tl = torch.zeros((K, max(s.p, 1)), dtype=torch.float64, device="cuda")
        tu = torch.zeros((K, s.n), dtype=torch.float64, device="cuda")
        s.set_trace(tl, tu, K)
    s.solve(alg, K, Kin)
    xl, xa, lam = s.result()
    out = dict(x_last=xl, x_avg=xa, lam=lam)
    if trace:
        out["trace_lam"] = tl.cpu().numpy()[:, :s.p]
        out["trace_u"] = tu.cpu().numpy()
    s.close()
    return out


def _dense_args(prob):
    return [prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone]


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("rho,alg", [(1.0, "DFGM"), (0.0, "DFGM"), (10.0, "DGM")])
def test_dense_sharded_bitwise_equals_single(torch_cuda, P, rho, alg):
    prob = qpgen.dense_ineq(1001, 333, seed=2)          # ragged: slices of unequal length
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, rho, 0.1)
    a = _run_sharded(torch_cuda, _dense_args(prob), P, rho, alg, 5, 6, L_in, L_d, trace=True)
    b = _run_single(torch_cuda, _dense_args(prob), rho, alg, 5, 6, L_in, L_d, trace=True)
    for k in ("x_last", "x_avg", "lam", "trace_lam", "trace_u"):
        assert np.array_equal(a[k], b[k]), (k, P)
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, alg, 5, 6, L_in, L_d)
    assert relerr(a["x_last"], r.x_last) <= 1e-9 and relerr(a["lam"], r.lam) <= 1e-9


@pytest.mark.parametrize("P", [2, 5])
def test_csr_sharded_bitwise_equals_single(torch_cuda, P):
    prob = qpgen.sparse_banded_eq(n=3001, p=1201, seed=4)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q.toarray(), prob.G.toarray(), 5.0, 0.5)
    args = [prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone]
    a = _run_sharded(torch_cuda, args, P, 5.0, "DFGM", 6, 5, L_in, L_d)
    b = _run_single(torch_cuda, args, 5.0, "DFGM", 6, 5, L_in, L_d)
    for k in ("x_last", "x_avg", "lam"):
        assert np.array_equal(a[k], b[k]), k


def test_more_ranks_than_constraint_rows(torch_cuda):
    """Degenerate shard: p < P leaves some ranks without G rows."""
    prob = qpgen.tiny(40, 3, seed=6, kind="mixed")
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.05)
    a = _run_sharded(torch_cuda, _dense_args(prob), 4, 1.0, "DFGM", 4, 3, L_in, L_d)
    b = _run_single(torch_cuda, _dense_args(prob), 1.0, "DFGM", 4, 3, L_in, L_d)
    for k in ("x_last", "x_avg", "lam"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.slow
def test_config2_full_size_8_way_sharding(torch_cuda):
    """BASELINE.json configs[2] at full size, 8-way row sharding (the 8-GPU layout) emulated on
    one GPU: bitwise equal to the 1-GPU solve on a 2 x 3 prefix."""
    d = qpgen.dense_ineq_torch(16384, 8192, seed=0, shift=0.05)
    args = [d[k] for k in ("Q", "q", "G", "g", "lb", "ub", "cone")]
    L_in, L_d = 47588.0, 1.0 / (1.0 + 0.05 / 47539.5)
    a = _run_sharded(torch_cuda, args, 8, 1.0, "DFGM", 2, 3, L_in, L_d, fused_path=False)
    b = _run_single(torch_cuda, args, 1.0, "DFGM", 2, 3, L_in, L_d)
    for k in ("x_last", "x_avg", "lam"):
        assert np.array_equal(a[k], b[k]), k
    # the row-sharded byte-floor step (default at this size) agrees with the two-pass solve
    c = _run_sharded(torch_cuda, args, 8, 1.0, "DFGM", 2, 3, L_in, L_d)
    for k in ("x_last", "x_avg", "lam"):
        assert relerr(c[k], b[k]) <= 1e-10, (k, relerr(c[k], b[k]))


@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("alg", ["DFGM", "DGM"])
def test_sharded_byte_floor_vs_oracle(torch_cuda, P, alg):
    """Row-sharded byte floor (n >= 4096, rho > 0): each rank streams the upper triangle of its Q
    rows and its G rows; the partial n-vectors are reduce-scattered (emulated: summed in rank order)
    -- against the oracle, and deterministic."""
    prob = qpgen.dense_ineq(4096, 2048, seed=1, shift=0.05)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.05)
    a = _run_sharded(torch_cuda, _dense_args(prob), P, 1.0, alg, 2, 4, L_in, L_d, trace=True)
    a2 = _run_sharded(torch_cuda, _dense_args(prob), P, 1.0, alg, 2, 4, L_in, L_d)
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, alg, 2, 4, L_in, L_d,
               keep_trace=True)
    for k, want in (("x_last", r.x_last), ("x_avg", r.x_avg), ("lam", r.lam)):
        assert relerr(a[k], want) <= 1e-9, (k, relerr(a[k], want))
        assert np.array_equal(a[k], a2[k])
    assert relerr(a["trace_u"], np.array(r.trace_u)) <= 1e-9


def test_sharded_byte_floor_ragged_warm_start_and_dual_average(torch_cuda):
    """Row-sharded byte floor on a ragged split (n = 4100 over 3 ranks, p = 1500 balanced against the
    slabs), warm-started, with the DGM dual-averaging final point -- against the oracle."""
    from paper_1504_05708_b200 import Solver, solve_emulated
    import torch
    prob = qpgen.dense_ineq(4100, 1500, seed=9, shift=0.05)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 2.0, 0.05)
    rng = np.random.default_rng(1)
    x0, lam0 = rng.uniform(-2, 2, 4100), np.abs(rng.standard_normal(1500))
    st = torch.cuda.Stream()
    ss = [Solver(*_dense_args(prob), rho=2.0, world_size=3, rank=r, emulate_ranks=True, stream=st.cuda_stream,
                 dual_average=True) for r in range(3)]
    prs = [s.p_range for s in ss]
    assert prs[0][0] == 0 and prs[-1][1] == 1500 and all(a[1] == b[0] for a, b in zip(prs, prs[1:]))
    assert prs[0][1] - prs[0][0] < prs[-1][1] - prs[-1][0]          # the first slab is the largest
    for s in ss:
        s.set_constants(L_in, L_d)
        s.set_initial(x0, lam0)
    solve_emulated(ss, "DGM", 3, 4)
    parts = [s.result() for s in ss]
    for s in ss:
        s.close()
    got = [np.concatenate([pt[i] for pt in parts]) for i in range(3)]
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 2.0, "DGM", 3, 4, L_in, L_d,
               x0=x0, lam0=lam0, dual_average=True)
    for g, w in zip(got, (r.x_last, r.x_avg, r.lam)):
        assert relerr(g, w) <= 1e-9, relerr(g, w)
