"""Batched MPC path (BASELINE.json configs[3]) vs the oracle (-m gpu).

The oracle runs the same DFOM on the n x B matrix of right-hand sides (each column one QP);
the GPU runs DMMA GEMMs with the fused epilogues.  Bar: 1e-9 relative per BASELINE.json.
"""
import numpy as np
import pytest

import qpgen
from oracle import dfom as O

pytestmark = pytest.mark.gpu
TOL = 1e-9


def relerr(got, want):
    got, want = np.asarray(got, float), np.asarray(want, float)
    return float(np.max(np.abs(got - want)) / (1.0 + np.max(np.abs(want)))) if want.size else 0.0


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _solve(prob, rho, alg, K, Kin, L_in, L_d, **kw):
    from paper_1504_05708_b200 import Solver
    s = Solver(prob.Q, prob.q.T.copy(), prob.G, prob.g.T.copy(), prob.lb, prob.ub, prob.cone, rho=rho, **kw)
    s.set_constants(L_in, L_d)
    info = s.solve(alg, K, Kin)
    xl, xa, lam = s.result()
    s.close()
    return xl, xa, lam, info


def _oracle(prob, rho, alg, K, Kin, L_in, L_d):
    return O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, alg, K, Kin, L_in, L_d)


@pytest.mark.parametrize("alg", ["DGM", "DFGM"])
@pytest.mark.parametrize("K,Kin", [(1, 1), (4, 6)])
def test_small_mpc_parity(torch_cuda, alg, K, Kin):
    prob = qpgen.mpc_batch(50, seed=2, N=4)          # n = 16, p = 96, B = 50 (ragged tiles)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    xl, xa, lam, _ = _solve(prob, 1.0, alg, K, Kin, L_in, L_d)
    r = _oracle(prob, 1.0, alg, K, Kin, L_in, L_d)
    assert relerr(xl, r.x_last.T) <= TOL and relerr(xa, r.x_avg.T) <= TOL and relerr(lam, r.lam.T) <= TOL


@pytest.mark.parametrize("B", [2, 37, 200])
def test_ragged_batches_and_rho0(torch_cuda, B):
    prob = qpgen.mpc_batch(B, seed=B, N=7)            # n = 28, p = 168
    for rho in (0.0, 2.0):
        L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, rho, 0.1)
        xl, xa, lam, _ = _solve(prob, rho, "DFGM", 5, 5, L_in, L_d)
        r = _oracle(prob, rho, O.DFGM, 5, 5, L_in, L_d)
        assert relerr(xl, r.x_last.T) <= TOL and relerr(xa, r.x_avg.T) <= TOL and relerr(lam, r.lam.T) <= TOL


def test_batched_equals_single_qp_solves(torch_cuda):
    """Each column of the batched solve equals the single-QP (GEMV) path on that QP
    (summation order differs only)."""
    from paper_1504_05708_b200 import Solver
    prob = qpgen.mpc_batch(6, seed=4, N=10)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    xl, xa, lam, _ = _solve(prob, 1.0, "DFGM", 6, 8, L_in, L_d)
    for b in range(6):
        s = Solver(prob.Q, prob.q[:, b], prob.G, prob.g[:, b], prob.lb, prob.ub, prob.cone, rho=1.0)
        s.set_constants(L_in, L_d)
        s.solve("DFGM", 6, 8)
        x1, a1, l1 = s.result()
        assert relerr(xl[b], x1) <= 1e-12 and relerr(lam[b], l1) <= 1e-12


def test_batch_sharding_is_exact(torch_cuda):
    """Batch-sharded multi-GPU mode (whole QPs per rank, no collective): ranks 0..2 of a
    3-way split solve disjoint QP slices whose concatenation is bitwise the 1-rank result."""
    from paper_1504_05708_b200 import Solver
    prob = qpgen.mpc_batch(70, seed=5, N=6)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    full = _solve(prob, 1.0, "DFGM", 5, 4, L_in, L_d)
    parts = []
    for rank in range(3):
        s = Solver(prob.Q, prob.q.T.copy(), prob.G, prob.g.T.copy(), prob.lb, prob.ub, prob.cone, rho=1.0,
                   world_size=3, rank=rank)
        s.set_constants(L_in, L_d)
        s.solve("DFGM", 5, 4)
        parts.append(s.result())
        s.close()
    for k in range(3):
        assert np.array_equal(np.concatenate([pt[k] for pt in parts]), full[k])


def test_lipschitz_on_batched_context(torch_cuda):
    from paper_1504_05708_b200 import Solver
    prob = qpgen.mpc_batch(16, seed=0)
    s = Solver(prob.Q, prob.q.T.copy(), prob.G, prob.g.T.copy(), prob.lb, prob.ub, prob.cone, rho=1.0,
               lambda_min_lb=0.1)
    L_in, L_d, nG2 = s.lipschitz(iters=120, safety=0.0)
    rL, rd, rn = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    assert abs(L_in - rL) <= 1e-9 * rL and abs(nG2 - rn) <= 1e-9 * rn and abs(L_d - rd) <= 1e-9 * rd


def test_config3_full_size_configured_counts(torch_cuda):
    """BASELINE.json configs[3] at full size: B = 8192 MPC QPs (n = 120, p = 720), DFGM rho = 1,
    50 x 20 (+20 last-iterate steps), in the bench launch configuration."""
    prob = qpgen.mpc_batch(8192, seed=0)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    xl, xa, lam, info = _solve(prob, 1.0, "DFGM", 50, 20, L_in, L_d)
    r = _oracle(prob, 1.0, O.DFGM, 50, 20, L_in, L_d)
    assert relerr(xl, r.x_last.T) <= TOL and relerr(xa, r.x_avg.T) <= TOL and relerr(lam, r.lam.T) <= TOL
    # paired rows (G = [Gamma; -Gamma]): [Q; Gamma] and Gamma' are streamed, 2B(n(n+P) + nP) flops,
    # P = 360, instead of the unpaired 2B(n(n+p) + np) = 3.067 GFLOP
    assert info["flops_pass_a"] + info["flops_pass_b"] == pytest.approx(2 * 8192 * (120 * 480 + 120 * 360), rel=1e-9)


def test_tall_blocks_both_passes(torch_cuda):
    """n = 132 > 128: pass B walks two 128-row blocks and pass A eight (M = 924, ragged last block);
    K = 160 / 800 after padding (several BK = 32 chunks through the ring)."""
    prob = qpgen.mpc_batch(45, seed=3, N=33)          # n = 132, p = 792
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    xl, xa, lam, _ = _solve(prob, 1.0, "DFGM", 3, 4, L_in, L_d)
    r = _oracle(prob, 1.0, O.DFGM, 3, 4, L_in, L_d)
    assert relerr(xl, r.x_last.T) <= TOL and relerr(xa, r.x_avg.T) <= TOL and relerr(lam, r.lam.T) <= TOL


_MULTI_GROUP = r"""
import sys, numpy as np
sys.path.insert(0, '.')
import qpgen
from oracle import dfom as O
from paper_1504_05708_b200 import Solver
prob = qpgen.mpc_batch(203, seed=7, N=33)
L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
s = Solver(prob.Q, prob.q.T.copy(), prob.G, prob.g.T.copy(), prob.lb, prob.ub, prob.cone, rho=1.0)
s.set_constants(L_in, L_d)
s.solve('DFGM', 3, 3)
got = s.result()
r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, 'DFGM', 3, 3, L_in, L_d)
err = max(float(np.max(np.abs(g - w.T)) / (1 + np.max(np.abs(w)))) for g, w in zip(got, (r.x_last, r.x_avg, r.lam)))
print('ERR', err)
"""


def test_several_groups_per_cta(torch_cuda):
    """Grid capped at 3 CTAs (DUQUAD_BATCHED_CTAS, read once per process, hence the subprocess):
    every CTA walks several QP groups through the same ring and mbarrier phases (203 QPs: 26
    octets; pass A 6 groups, pass B 9 groups, ragged last octet)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, DUQUAD_BATCHED_CTAS="3")
    out = subprocess.run([sys.executable, "-c", _MULTI_GROUP], env=env, capture_output=True, text=True,
                         timeout=600, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0, out.stderr[-2000:]
    err = float(out.stdout.split("ERR")[-1])
    assert err <= TOL, err


@pytest.mark.parametrize("alg", ["DGM", "DFGM"])
def test_paired_rows_match_unpaired_and_detection(torch_cuda, alg):
    """pair_rows: G = [Gamma; -Gamma] runs the reduced matrices ([Q; Gamma] in pass A, Gamma'(w_top -
    w_bottom) in pass B); the iterates equal the unpaired kernels' to rounding (1e-12) and the
    oracle's (1e-9), incl. the DFOM step and DGM dual averaging.  A G whose halves are not exact
    negatives (one entry off by 1 ulp) is not paired."""
    prob = qpgen.mpc_batch(77, seed=8, N=9)              # n = 36, p = 216, P = 108
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    n, p, B = 36, 216, 77
    kw = dict(dual_average=True) if alg == "DGM" else {}
    a = _solve(prob, 1.0, alg, 6, 5, L_in, L_d, **kw)
    b = _solve(prob, 1.0, alg, 6, 5, L_in, L_d, pair_rows=False, **kw)
    assert a[3]["flops_pass_a"] == pytest.approx(2.0 * (n + p // 2) * n * B)
    assert b[3]["flops_pass_a"] == pytest.approx(2.0 * (n + p) * n * B)
    for k in range(3):
        assert relerr(a[k], b[k]) <= 1e-12, k
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, alg, 6, 5, L_in, L_d,
               dual_average=alg == "DGM")
    assert relerr(a[0], r.x_last.T) <= TOL and relerr(a[1], r.x_avg.T) <= TOL and relerr(a[2], r.lam.T) <= TOL
    G = prob.G.copy()
    G[p // 2 + 3, 5] = np.nextafter(G[p // 2 + 3, 5], np.inf)
    prob.G = G
    c = _solve(prob, 1.0, alg, 2, 2, L_in, L_d, **kw)
    assert c[3]["flops_pass_a"] == pytest.approx(2.0 * (n + p) * n * B)


@pytest.mark.parametrize("seed", range(5))
def test_random_batched_shapes(torch_cuda, seed):
    """Randomised batch sizes and horizons for the persistent DMMA kernels: ragged octets, n across
    the 128-row block boundary, p with ragged 32-column chunks."""
    rng = np.random.default_rng(300 + seed)
    B = int(rng.integers(2, 260))
    N = int([2, 9, 31, 33, 40][seed])                  # n = 4N: 8 ... 160
    prob = qpgen.mpc_batch(B, seed=seed, N=N)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    r = _oracle(prob, 1.0, O.DFGM, 2, 3, L_in, L_d)
    for pair in (True, False):
        xl, xa, lam, info = _solve(prob, 1.0, "DFGM", 2, 3, L_in, L_d, pair_rows=pair)
        assert info["path"] == 4
        assert relerr(xl, r.x_last.T) <= TOL and relerr(xa, r.x_avg.T) <= TOL and relerr(lam, r.lam.T) <= TOL
