"""Byte-floor inner step (symmetric-Q triangle + single G read, CTA-pair clusters) vs the oracle
and vs the two-pass path (-m gpu)."""
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


def _solve(torch, prob, rho, alg, K, Kin, L_in, L_d, fused=True, trace=False):
    from paper_1504_05708_b200 import Solver
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=rho, fused_path=fused)
    s.set_constants(L_in, L_d)
    if trace:
        tl = torch.zeros((K, max(prob.p, 1)), dtype=torch.float64, device="cuda")
        tu = torch.zeros((K, prob.n), dtype=torch.float64, device="cuda")
        s.set_trace(tl, tu, K)
    info = s.solve(alg, K, Kin)
    xl, xa, lam = s.result()
    out = dict(x_last=xl, x_avg=xa, lam=lam, info=info)
    if trace:
        out["trace_lam"] = tl.cpu().numpy()[:, :prob.p]
        out["trace_u"] = tu.cpu().numpy()
    s.close()
    return out


@pytest.fixture(scope="module")
def probs():
    return {"4096": qpgen.dense_ineq(4096, 2048, seed=1, shift=0.05),
            "ragged": qpgen.tiny(5000, 3001, seed=2, kind="mixed", shift=0.05)}


@pytest.mark.parametrize("name", ["4096", "ragged"])
@pytest.mark.parametrize("rho,alg", [(1.0, "DFGM"), (1.0, "DGM"), (0.0, "DFGM"), (4.0, "DFGM")])
def test_fused_matches_oracle_and_two_pass(torch_cuda, probs, name, rho, alg):
    prob = probs[name]
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, rho, 0.05)
    K, Kin = 4, 5
    a = _solve(torch_cuda, prob, rho, alg, K, Kin, L_in, L_d, fused=True, trace=True)
    b = _solve(torch_cuda, prob, rho, alg, K, Kin, L_in, L_d, fused=False, trace=True)
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, alg, K, Kin, L_in, L_d,
               keep_trace=True)
    for k, want in (("x_last", r.x_last), ("x_avg", r.x_avg), ("lam", r.lam)):
        assert relerr(a[k], want) <= TOL, (k, relerr(a[k], want))
        assert relerr(a[k], b[k]) <= 1e-12, k
    for j in range(K):
        assert relerr(a["trace_lam"][j], r.trace_lam[j]) <= TOL
        assert relerr(a["trace_u"][j], r.trace_u[j]) <= TOL
    # fewer bytes per step than the two-pass path
    assert a["info"]["bytes_pass_a"] + a["info"]["bytes_pass_b"] < 0.8 * (
        b["info"]["bytes_pass_a"] + b["info"]["bytes_pass_b"])


def test_fused_no_constraints(torch_cuda):
    prob = qpgen.tiny(4100, 0, seed=3, shift=0.05)
    L_in, _, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.05)
    a = _solve(torch_cuda, prob, 1.0, "DFGM", 3, 6, L_in, 1.0)
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, "DFGM", 3, 6, L_in, 1.0)
    assert relerr(a["x_last"], r.x_last) <= TOL and relerr(a["x_avg"], r.x_avg) <= TOL


def test_fused_is_deterministic(torch_cuda, probs):
    prob = probs["4096"]
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.05)
    a = _solve(torch_cuda, prob, 1.0, "DFGM", 3, 4, L_in, L_d)
    b = _solve(torch_cuda, prob, 1.0, "DFGM", 3, 4, L_in, L_d)
    for k in ("x_last", "x_avg", "lam"):
        assert np.array_equal(a[k], b[k])


@pytest.mark.slow
def test_fused_config2_full_size(torch_cuda):
    """configs[2] at full size through the byte-floor step (the bench's launch configuration)."""
    from paper_1504_05708_b200 import Solver
    d = qpgen.dense_ineq_torch(16384, 8192, seed=0, shift=0.05)
    s = Solver(d["Q"], d["q"], d["G"], d["g"], d["lb"], d["ub"], d["cone"], rho=1.0, lambda_min_lb=0.05)
    L_in, L_d, _ = s.lipschitz(iters=60, safety=1e-3)
    s.solve("DFGM", 2, 3)
    xl, xa, lam = s.result()
    h = {k: v.cpu().numpy() for k, v in d.items()}
    r = O.dfom(h["Q"], h["q"], h["G"], h["g"], h["lb"], h["ub"], h["cone"], 1.0, O.DFGM, 2, 3, L_in, L_d)
    assert relerr(xl, r.x_last) <= TOL and relerr(xa, r.x_avg) <= TOL and relerr(lam, r.lam) <= TOL
    s.close()


def test_fused_mixed_cones_ragged_infinite_bounds(torch_cuda):
    """Byte floor on a ragged n = 4103 with alternating equality / inequality rows and a box that is
    infinite on some coordinates."""
    from paper_1504_05708_b200 import Solver
    prob = qpgen.tiny(4103, 1001, seed=21, kind="mixed", shift=0.1)
    prob.lb[::5] = -np.inf
    prob.ub[1::7] = np.inf
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0)
    s.set_constants(L_in, L_d)
    assert s.solve("DFGM", 2, 3)["path"] == 1
    got = s.result()
    s.close()
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, "DFGM", 2, 3, L_in, L_d)
    for g, w in zip(got, (r.x_last, r.x_avg, r.lam)):
        assert relerr(g, w) <= 1e-9, relerr(g, w)


@pytest.mark.parametrize("seed", range(6))
def test_fused_random_shapes_match_two_pass(torch_cuda, seed):
    """Randomised shapes for the byte floor's partitioning (ragged tile columns, Q pieces, G pairs
    and column blocks): n in [4096, 8200], p from 0 / a handful of rows to > n / 2, mixed cones --
    against the two-pass path on the same problem (different summation order: 1e-11)."""
    from paper_1504_05708_b200 import Solver
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(4096, 8200))
    p = int([0, 1, 3, int(rng.integers(5, 300)), int(rng.integers(300, n // 2)), int(rng.integers(n // 2, n))][seed])
    prob = qpgen.tiny(n, max(p, 1), seed=seed, kind="mixed", shift=0.2)
    if p == 0:
        prob.G, prob.g, prob.cone = prob.G[:0], prob.g[:0], prob.cone[:0]
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.2) if p else (
        float(np.linalg.eigvalsh(prob.Q).max()) * 1.01, 0.0, 0.0)
    out = []
    for fused in (True, False):
        s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0, fused_path=fused,
                   eq_precompute=False)
        s.set_constants(L_in, L_d)
        info = s.solve("DFGM", 2, 3)
        assert (info["path"] == 1) == fused, (info["path"], fused)
        out.append(s.result())
        s.close()
    for a, b in zip(*out):
        assert relerr(a, b) <= 1e-11, (n, p, relerr(a, b))
