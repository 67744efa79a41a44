"""Multi-process (world_size 2, gloo, CPU) tests of the N > 1 host logic (-m "not gpu").

* the NCCL unique id travels from rank 0 to every rank through torch.distributed, exactly as
  bench.py does it (a 128-byte blob; generated here without NCCL);
* the row partition from the C library (duquad_shard_range) tiles every matrix on every rank;
* the decomposition the sharded kernels implement -- rank r owns rows R_r of Q, S_r of G and R_r
  of G'; replicas of y (n) and w (p) refreshed by an all-gather after each pass; the DFOM dual
  update and the primal average row-local -- reproduces the unsharded oracle: a per-rank NumPy
  model of that schedule, with gloo all_gather as the exchange, is compared with oracle.dfom.
"""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker_id(rank, world, port, q):
    _init(rank, world, port)
    import sys
    sys.path.insert(0, ROOT)
    blob = [os.urandom(128) if rank == 0 else None]
    dist.broadcast_object_list(blob, src=0)
    from paper_1504_05708_b200 import shard_range
    rng = [shard_range(n, world, rank) for n in (16384, 8192, 1001, 333, 3)]
    q.put((rank, blob[0], rng))
    dist.destroy_process_group()


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_id_broadcast_and_partition():
    from paper_1504_05708_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_id, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=120) for _ in ps])
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == res[1][1] and len(res[0][1]) == 128
    for i, n in enumerate((16384, 8192, 1001, 333, 3)):
        (b0, e0), (b1, e1) = res[0][2][i], res[1][2][i]
        assert b0 == 0 and e0 == b1 and e1 == n


def _sharded_dfom(rank, world, port, q, K, Kin, rho, alg):
    """Per-rank model of the kernels' schedule (capi.cu outer_phase), gloo all-gathers."""
    _init(rank, world, port)
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import qpgen
    from oracle import dfom as O
    prob = qpgen.dense_ineq(61, 23, seed=11)
    n, p = prob.n, prob.p
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, rho, 0.1)
    ns, ps = -(-n // world), -(-p // world)
    R = slice(min(n, rank * ns), min(n, (rank + 1) * ns))
    S = slice(min(p, rank * ps), min(p, (rank + 1) * ps))
    Qr, Gr, GTr = prob.Q[R], prob.G[S], prob.G.T[R]
    cone = prob.cone[S]

    def allgather(local, slice_len, total):
        buf = np.zeros(slice_len)
        buf[:len(local)] = local
        out = [torch.zeros(slice_len, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, torch.from_numpy(buf))
        return np.concatenate([o.numpy() for o in out])[:total]

    th = O.theta_sequence(K + 2)
    bin_ = O.beta_fgm(Kin)
    x = O.clamp_U(np.zeros(n), prob.lb, prob.ub)[R]
    y_full = allgather(x, ns, n)
    mu = np.zeros(S.stop - S.start)
    lam_prev = np.zeros_like(mu)
    xhat = np.zeros_like(x)
    S_acc = 0.0
    for j in range(1, K + 2):
        last = j == K + 1
        for k in range(1, Kin + 1):
            r = Gr @ y_full + prob.g[S]                       # pass A, G rows
            Qy = Qr @ y_full                                   # pass A, Q rows
            if k == 1 and j >= 2:                              # fused DFOM step (row-local)
                s = O.slack(r, mu, cone, rho)
                lam = O.proj_Kd(mu + (0.5 / L_d) * (r - s), cone, True)
                b = 0.0 if (last or alg == O.DGM) else (th[j - 1] - 1.0) / th[j]
                mu = lam + b * (lam - lam_prev)
                lam_prev = lam
            w = rho * ((r + mu / rho) - O.proj_K(r + mu / rho, cone)) if rho > 0 else mu
            w_full = allgather(w, ps, p)                       # all-gather w
            grad = Qy + prob.q[R] + GTr @ w_full               # pass B
            xn = O.clamp_U(y_full[R] - grad / L_in, prob.lb[R], prob.ub[R])
            yn = xn if k == Kin else xn + bin_[k] * (xn - x)
            x = xn
            if k == Kin and not last:                          # running average (row-local)
                om = th[j] if alg == O.DFGM else 1.0
                S_acc += om
                xhat = xhat + (om / S_acc) * (x - xhat)
            y_full = allgather(yn, ns, n)                      # all-gather y
    q.put((rank, x, xhat, lam_prev))
    dist.destroy_process_group()


@pytest.mark.parametrize("rho,alg", [(1.0, "DFGM"), (0.0, "DGM")])
def test_row_sharded_schedule_reproduces_oracle(rho, alg):
    import qpgen
    from oracle import dfom as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    K, Kin = 6, 5
    ps = [ctx.Process(target=_sharded_dfom, args=(r, 2, port, q, K, Kin, rho, alg)) for r in range(2)]
    for p in ps:
        p.start()
    parts = sorted([q.get(timeout=300) for _ in ps], key=lambda t: t[0])
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = np.concatenate([t[1] for t in parts])
    xh = np.concatenate([t[2] for t in parts])
    lam = np.concatenate([t[3] for t in parts])
    prob = qpgen.dense_ineq(61, 23, seed=11)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, rho, 0.1)
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, alg, K, Kin, L_in, L_d)
    assert np.allclose(x, r.x_last, rtol=0, atol=1e-12)
    assert np.allclose(xh, r.x_avg, rtol=0, atol=1e-12)
    assert np.allclose(lam, r.lam, rtol=0, atol=1e-12)
