"""The row-sharded code path with REAL NCCL collectives on one GPU (option nccl_self, -m gpu).

A P-GPU run cannot be launched here (gpurun and the round-end tiers have one GPU, and NCCL
refuses two ranks on one device), and the emulated-rank tests replace the collectives with device
copies.  nccl_self runs a world-size-1 context on the row-sharded code path over a one-rank NCCL
communicator, so every collective a P-GPU run issues -- the y / w all-gathers, the grouped w
broadcasts, the byte floor's reduce-scatter, the eps_in all-reduce and the Lipschitz power
iteration's all-reduces -- is called with the same buffers and counts (P = 1), inside the same
CUDA-graph captures, on real NCCL.  Results must match the oracle (1e-9) and, where the row sums
are the single-GPU ones (two-pass, CSR), the plain world-1 solve bit for bit."""
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


def _solve(prob, rho, alg, K, Kin, L_in, L_d, **kw):
    from paper_1504_05708_b200 import Solver
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=rho, **kw)
    s.set_constants(L_in, L_d)
    info = s.solve(alg, K, Kin)
    out = s.result()
    s.close()
    return info, out


def _oracle(prob, rho, alg, K, Kin, L_in, L_d):
    return O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, alg, K, Kin, L_in, L_d)


@pytest.mark.parametrize("use_graphs", [True, False])
@pytest.mark.parametrize("alg", ["DGM", "DFGM"])
def test_two_pass_allgathers_bitwise(torch_cuda, alg, use_graphs):
    prob = qpgen.tiny(301, 97, seed=6, kind="mixed", shift=0.2)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.2)
    kw = dict(small_path=False, fused_path=False, use_graphs=use_graphs)
    info, (xl, xa, lam) = _solve(prob, 1.0, alg, 5, 6, L_in, L_d, nccl_self=True, **kw)
    _, ref = _solve(prob, 1.0, alg, 5, 6, L_in, L_d, **kw)
    for a, b in zip((xl, xa, lam), ref):
        assert np.array_equal(a, b)
    r = _oracle(prob, 1.0, alg, 5, 6, L_in, L_d)
    for got, want in ((xl, r.x_last), (xa, r.x_avg), (lam, r.lam)):
        assert relerr(got, want) <= TOL


@pytest.mark.parametrize("rho", [1.0, 0.0])
def test_byte_floor_reduce_scatter(torch_cuda, rho):
    """n >= 4096, rho > 0: the row-sharded byte floor (partial n-vector -> ncclReduceScatter ->
    k_slice_epi -> y all-gather); rho = 0: the sharded K3 path's all-gathers."""
    prob = qpgen.dense_ineq(4100, 1500, seed=3, shift=0.1)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, rho, 0.1)
    info, (xl, xa, lam) = _solve(prob, rho, "DFGM", 2, 4, L_in, L_d, nccl_self=True)
    r = _oracle(prob, rho, "DFGM", 2, 4, L_in, L_d)
    for got, want in ((xl, r.x_last), (xa, r.x_avg), (lam, r.lam)):
        assert relerr(got, want) <= TOL, relerr(got, want)


def test_csr_bitwise(torch_cuda):
    prob = qpgen.sparse_banded_eq(n=3001, p=1201, seed=4)
    Qd, Gd = prob.Q.toarray(), prob.G.toarray()
    L_in, L_d, _ = O.lipschitz_constants(Qd, Gd, 5.0, 0.5)
    _, got = _solve(prob, 5.0, "DFGM", 4, 5, L_in, L_d, nccl_self=True)
    _, ref = _solve(prob, 5.0, "DFGM", 4, 5, L_in, L_d)
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)


def test_eps_mode_allreduce(torch_cuda):
    """eps_in mode: the stop test's sum goes through ncclAllReduce before k_inner_decide; with one
    rank the decisions (and so the counts and iterates) are the world-1 ones, on both the two-pass
    and the sharded byte-floor schedule."""
    from paper_1504_05708_b200 import Solver
    for n, p, kw in ((301, 97, dict(small_path=False, fused_path=False)), (4100, 1500, {})):
        prob = qpgen.dense_ineq(n, p, seed=3, shift=0.1)
        prob.G *= 0.05
        prob.g *= 0.05
        L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
        outs = []
        for ns in (True, False):
            s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0, nccl_self=ns, **kw)
            s.set_constants(L_in, L_d)
            info = s.solve_eps("DFGM", 3, 120, 1e-4, 0.1)
            outs.append((info["inner_counts"], s.result()))
            s.close()
        assert outs[0][0] == outs[1][0] and any(c < 120 for c in outs[0][0])
        r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, "DFGM", 3, outs[0][0],
                   L_in, L_d)
        xl, xa, lam = outs[0][1]
        for got, want in ((xl, r.x_last), (xa, r.x_avg), (lam, r.lam)):
            assert relerr(got, want) <= TOL, (n, relerr(got, want))


def test_lipschitz_allreduce(torch_cuda):
    """The power / Lanczos iteration's dot products are all-reduced over the ranks: with one rank
    the estimates are the world-1 ones."""
    from paper_1504_05708_b200 import Solver
    prob = qpgen.tiny(301, 97, seed=6, kind="mixed", shift=0.2)
    est = []
    for ns in (True, False):
        s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0, nccl_self=ns,
                   small_path=False, fused_path=False)
        est.append(s.lipschitz(60))
        s.close()
    assert np.allclose(np.asarray(est[0], float), np.asarray(est[1], float), rtol=1e-12, atol=0)


def test_state_resume_and_warm_start(torch_cuda):
    """get_state / set_state and set_initial on the nccl_self path: resume is bitwise the
    uninterrupted solve; a warm start matches the oracle from the same start."""
    from paper_1504_05708_b200 import Solver
    prob = qpgen.tiny(301, 97, seed=6, kind="mixed", shift=0.2)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.2)
    mk = lambda: Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0, nccl_self=True,
                        small_path=False, fused_path=False, checkpoint=True)
    a = mk()
    a.set_constants(L_in, L_d)
    a.solve("DFGM", 5, 6)
    full = a.result()
    b = mk()
    b.set_constants(L_in, L_d)
    b.solve("DFGM", 2, 6)
    st = b.get_state()
    c = mk()
    c.set_constants(L_in, L_d)
    c.set_state(st)
    c.solve("DFGM", 3, 6)
    for x, y in zip(c.result(), full):
        assert np.array_equal(x, y)
    rng = np.random.default_rng(7)
    x0 = rng.uniform(-2.0, 2.0, prob.n)
    lam0 = np.abs(rng.standard_normal(prob.p))
    a.set_initial(x0, lam0)
    a.solve("DFGM", 4, 5)
    xl, xa, lam = a.result()
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, "DFGM", 4, 5, L_in, L_d,
               x0=x0, lam0=lam0)
    for got, want in ((xl, r.x_last), (xa, r.x_avg), (lam, r.lam)):
        assert relerr(got, want) <= TOL
    for s in (a, b, c):
        s.close()


_PROBE = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import qpgen
from paper_1504_05708_b200 import Solver
prob = qpgen.dense_ineq(int(sys.argv[2]), int(sys.argv[3]), seed=3, shift=0.1)
s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0, nccl_self=True,
           small_path=False, fused_path=sys.argv[4] == "1")
s.set_constants(50.0, 1.0)
info = s.solve("DFGM", 2, 3)
print("PATH", info["path"], flush=True)
print("LIP", s.lipschitz(5), "RES", s.residuals(), flush=True)   # w replica + all-reduced dots
s.close()
"""


@pytest.mark.parametrize("n,p,fused,need", [(301, 97, "0", ("AllGather", "AllReduce")),
                                            (4100, 1500, "1", ("AllGather", "ReduceScatter", "Broadcast",
                                                                        "AllReduce"))])
def test_collectives_are_really_issued(torch_cuda, n, p, fused, need):
    """NCCL's own log (NCCL_DEBUG_SUBSYS=COLL) shows the collectives the sharded schedule issues:
    the y / w all-gathers on the two-pass path; on the byte floor the reduce-scatter, the y
    all-gathers and (Lanczos / residuals) the grouped broadcasts of the balanced w replica; the
    all-reduced dot products on both."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="COLL")
    out = subprocess.run([sys.executable, "-c", _PROBE, root, str(n), str(p), fused], env=env, cwd=root,
                         capture_output=True, text=True, timeout=300)
    log = out.stdout + out.stderr
    assert out.returncode == 0, log[-3000:]
    assert ("PATH 1" in log) == (fused == "1"), log[-2000:]
    for op in need:
        assert f"{op}: opCount" in log, (op, log[-3000:])
