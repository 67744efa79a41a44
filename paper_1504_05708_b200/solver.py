"""Thin Python binding over the DuQuad C ABI (include/duquad.h).

Marshalling only: every step of the solve runs in the library's sm_100a
kernels.  Inputs may be NumPy arrays (host) or torch tensors (host or CUDA);
torch is used for nothing but device memory, streams and process groups.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib as L

_ALGS = {"DGM": L.DGM, "DFGM": L.DFGM}
_INNER = {"FGM": L.INNER_FGM, "GM": L.INNER_GM, "FGM_SIGMA": L.INNER_FGM_SIGMA}


def _is_torch(x):
    return type(x).__module__.startswith("torch")


class _Arr:
    """Keeps a contiguous fp64/uint8/int32 buffer alive and exposes its address."""

    def __init__(self, x, dtype):
        if x is None:
            self.obj, self.ptr, self.dev = None, None, False
            return
        if _is_torch(x):
            import torch
            tdt = {np.float64: torch.float64, np.uint8: torch.uint8, np.int32: torch.int32}[dtype]
            t = x.detach()
            if t.dtype != tdt:
                t = t.to(tdt)
            t = t.contiguous()
            self.obj, self.ptr, self.dev = t, t.data_ptr(), t.is_cuda
        else:
            a = np.ascontiguousarray(x, dtype=dtype)
            self.obj, self.ptr, self.dev = a, a.ctypes.data, False


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    L.check(L.lib().duquad_nccl_unique_id(buf))
    return buf.raw


def shard_range(rows: int, world: int, rank: int):
    b, e = C.c_int64(), C.c_int64()
    L.check(L.lib().duquad_shard_range(rows, world, rank, C.byref(b), C.byref(e)))
    return b.value, e.value


def solve_emulated(solvers, alg: str = "DFGM", outer: int = 1, inner: int = 1):
    """Runs P row-sharded Solvers (ranks 0..P-1, emulate_ranks=True, same device and stream) in
    lock step on one GPU; all-gathers are device copies (testing the sharded path, row a11)."""
    arr = (C.c_void_p * len(solvers))(*[s._ctx.value for s in solvers])
    L.check(L.lib().duquad_solve_emulated(arr, len(solvers), _ALGS[alg], int(outer), int(inner)),
            solvers[0]._ctx)


def solve_emulated_eps(solvers, alg: str, outer: int, inner_max: int, eps_in: float, sigma_L: float) -> dict:
    """solve_emulated with eps_in-driven inner stopping (duquad_solve_eps_emulated): the stop test's
    sum is all-reduced over the ranks (emulated: added in rank order), so every rank takes the same
    decision.  Returns the per-solve counts / converged flags (identical on every rank)."""
    arr = (C.c_void_p * len(solvers))(*[s._ctx.value for s in solvers])
    st = L.lib().duquad_solve_eps_emulated(arr, len(solvers), _ALGS[alg], int(outer), int(inner_max), float(eps_in),
                                           float(sigma_L))
    if st not in (L.DUQUAD_OK, L.DUQUAD_EMAXITER):
        L.check(st, solvers[0]._ctx)
    m = int(outer) + 1
    out = []
    for s in solvers:
        counts, conv = (C.c_int32 * m)(), (C.c_int32 * m)()
        L.check(L.lib().duquad_get_inner_counts(s._ctx, counts, conv, m), s._ctx)
        out.append((list(counts), [bool(c) for c in conv]))
    assert all(o == out[0] for o in out), "ranks disagree on the stop decisions"
    return dict(inner_counts=out[0][0], converged=out[0][1], capped=st == L.DUQUAD_EMAXITER)


def theory_schedule(alg: str, eps: float, R_d: float, L_d: float, L_in: float, sigma_L: float, D_U: float,
                    normG: float, lambda_min_Q: float = 0.0, lambda_max_Q: float = 0.0) -> dict:
    """DuQuad's theory schedule (include/duquad.h duquad_theory_schedule; host arithmetic).
    case_id 1 iff lambda_min_Q > 1e-7 max(1, lambda_max_Q) (SPEC.md:186's tau_pd)."""
    out = L.Schedule()
    L.check(L.lib().duquad_theory_schedule(_ALGS[alg], float(eps), float(R_d), float(L_d), float(L_in),
                                           float(sigma_L), float(D_U), float(normG), float(lambda_min_Q),
                                           float(lambda_max_Q),
                                           C.byref(out)))
    return {k: getattr(out, k) for k, _ in L.Schedule._fields_ if k != "reserved"}


def theory_bounds(alg: str, k: int, L_d: float, R_d: float, eps_in: float) -> dict:
    """Convergence-bound diagnostics after k outer iterations (include/duquad.h duquad_theory_bounds)."""
    out = L.Bounds()
    L.check(L.lib().duquad_theory_bounds(_ALGS[alg], int(k), float(L_d), float(R_d), float(eps_in),
                                         C.byref(out)))
    return {k_: getattr(out, k_) for k_, _ in L.Bounds._fields_}


class Solver:
    """One DuQuad context: setup (pack + upload), constants, solve, results.

    Q (n x n), q (n), G (p x n), g (p), lb, ub (n), cone (p uint8: 0 ZERO, 1 NONPOS)
    follow PAPER.md:193-212.  All float inputs must be fp64 (converted otherwise).
    """

    def __init__(self, Q, q, G, g, lb, ub, cone=None, rho: float = 1.0, *,
                 dual_step_scale: float = 0.5, project_dual: bool = True, inner_rule: str = "FGM",
                 sigma: float = 0.0, lambda_min_lb: float = 0.0, l_mode: int = 0,
                 use_graphs: bool = True, world_size: int = 1, rank: int = 0,
                 nccl_id: Optional[bytes] = None, stream=None, device: int = -1,
                 time_passes: bool = False, cone_all: int = L.CONE_NONPOS, small_path: bool = True,
                 rho0_path: bool = True, emulate_ranks: bool = False, fused_path: bool = True,
                 persist_path: bool = False, dual_average: bool = False, eq_precompute: bool = True,
                 checkpoint: bool = False, nccl_self: bool = False, sell_path: bool = True,
                 pair_rows: bool = True, pdl: bool = True):
        """Dense Q (n x n) and G (p x n), or scipy.sparse matrices (-> CSR path, row a10).
        dual_average: DGM final dual point from the average of lambda^0..lambda^K.
        nccl_self: world_size 1 on the row-sharded code path over a one-rank NCCL communicator.
        sell_path: CSR input with short rows runs lane-per-row kernels (SELL-32 / thread-per-row).
        pair_rows: batched QPs with G = [G_t; -G_t] stream G_t only (half the G work).
        pdl: programmatic dependent launch of the inner-step kernels."""
        if hasattr(Q, "tocsr"):
            Qc = Q.tocsr()
            Qc.sort_indices()
            Gc = G.tocsr()
            Gc.sort_indices()
            arrs = dict(Q_rowptr=_Arr(Qc.indptr, np.int32), Q_col=_Arr(Qc.indices, np.int32),
                        Q_val=_Arr(Qc.data, np.float64), G_rowptr=_Arr(Gc.indptr, np.int32),
                        G_col=_Arr(Gc.indices, np.int32), G_val=_Arr(Gc.data, np.float64))
            n, p = Qc.shape[0], Gc.shape[0]
            fmt, nnz = L.CSR, (Qc.nnz, Gc.nnz)
        else:
            arrs = dict(Q=_Arr(Q, np.float64), G=_Arr(G, np.float64))
            n = int(arrs["Q"].obj.shape[0])
            p = int(arrs["G"].obj.shape[0]) if arrs["G"].obj is not None else 0
            fmt, nnz = L.DENSE, (0, 0)
        self._init(arrs, fmt, n, p, nnz, q, g, lb, ub, cone, rho, cone_all,
                   dict(dual_step_scale=dual_step_scale, project_dual=project_dual, inner_rule=inner_rule,
                        sigma=sigma, lambda_min_lb=lambda_min_lb, l_mode=l_mode, use_graphs=use_graphs,
                        world_size=world_size, rank=rank, nccl_id=nccl_id, stream=stream, device=device,
                        time_passes=time_passes, small_path=small_path, rho0_path=rho0_path,
                        emulate_ranks=emulate_ranks, fused_path=fused_path, persist_path=persist_path,
                        dual_average=dual_average, eq_precompute=eq_precompute, checkpoint=checkpoint,
                        nccl_self=nccl_self, sell_path=sell_path, pair_rows=pair_rows, pdl=pdl))

    @classmethod
    def csr(cls, n, p, Q_rowptr, Q_col, Q_val, G_rowptr, G_col, G_val, q, g, lb, ub, cone=None,
            rho: float = 1.0, cone_all: int = L.CONE_ZERO, **opts):
        """CSR problem from raw arrays (NumPy on the host or torch on the device; int32 indices)."""
        self = cls.__new__(cls)
        arrs = dict(Q_rowptr=_Arr(Q_rowptr, np.int32), Q_col=_Arr(Q_col, np.int32), Q_val=_Arr(Q_val, np.float64),
                    G_rowptr=_Arr(G_rowptr, np.int32), G_col=_Arr(G_col, np.int32), G_val=_Arr(G_val, np.float64))
        nnz = (int(arrs["Q_val"].obj.shape[0]), int(arrs["G_val"].obj.shape[0]))
        defaults = dict(dual_step_scale=0.5, project_dual=True, inner_rule="FGM", sigma=0.0, lambda_min_lb=0.0,
                        l_mode=0, use_graphs=True, world_size=1, rank=0, nccl_id=None, stream=None, device=-1,
                        time_passes=False, small_path=True)
        defaults.update(opts)
        self._init(arrs, L.CSR, int(n), int(p), nnz, q, g, lb, ub, cone, rho, cone_all, defaults)
        return self

    def _init(self, arrs, fmt, n, p, nnz, q, g, lb, ub, cone, rho, cone_all, o):
        lib = L.lib()
        self._lib = lib
        arrs.update(q=_Arr(q, np.float64), g=_Arr(g, np.float64), lb=_Arr(lb, np.float64),
                    ub=_Arr(ub, np.float64), cone=_Arr(cone, np.uint8))
        devs = {k: a.dev for k, a in arrs.items() if a.obj is not None and getattr(a.obj, "size", 1) != 0}
        if len(set(devs.values())) > 1:
            raise ValueError("problem arrays must be all on the host or all on the device")
        on_device = bool(devs and next(iter(devs.values())))
        # batched mode (row a9): q is B x n and g is B x p (row b = QP b), Q and G shared
        qshape = tuple(arrs["q"].obj.shape)
        batch = int(qshape[0]) if len(qshape) == 2 else 1
        if batch > 1 and tuple(arrs["g"].obj.shape) != (batch, p):
            raise ValueError("batched g must be B x p")
        prob = L.Problem()
        prob.n, prob.p, prob.batch = n, p, batch
        prob.format = fmt
        prob.on_device = int(on_device)
        for k, a in arrs.items():
            setattr(prob, k, a.ptr)
        prob.ldQ = prob.ldG = n
        prob.Q_nnz, prob.G_nnz = nnz
        prob.cone_all = cone_all
        opt = L.Options()
        lib.duquad_default_options(C.byref(opt))
        opt.dual_step_scale = o["dual_step_scale"]
        opt.project_dual = int(o["project_dual"])
        opt.inner_rule = _INNER[o["inner_rule"]]
        opt.sigma = o["sigma"]
        opt.lambda_min_lb = o["lambda_min_lb"]
        opt.l_mode = o["l_mode"]
        opt.use_graphs = int(o["use_graphs"])
        opt.world_size = o["world_size"]
        opt.rank = o["rank"]
        nid = o["nccl_id"]
        self._nccl_id = C.create_string_buffer(nid, 128) if nid is not None else None
        opt.nccl_id = C.cast(self._nccl_id, C.c_void_p) if self._nccl_id is not None else None
        opt.stream = o["stream"]
        opt.device = o["device"]
        opt.time_passes = int(o["time_passes"])
        opt.small_path = int(o.get("small_path", True))
        opt.rho0_path = int(o.get("rho0_path", True))
        opt.emulate_ranks = int(o.get("emulate_ranks", False))
        opt.fused_path = int(o.get("fused_path", True))
        opt.persist_path = int(o.get("persist_path", False))
        opt.dual_average = int(o.get("dual_average", False))
        opt.eq_precompute = int(o.get("eq_precompute", True))
        opt.checkpoint = int(o.get("checkpoint", False))
        opt.nccl_self = int(o.get("nccl_self", False))
        opt.sell_path = int(o.get("sell_path", True))
        opt.pair_rows = int(o.get("pair_rows", True))
        opt.pdl = int(o.get("pdl", True))
        ctx = C.c_void_p()
        L.check(lib.duquad_setup(C.byref(ctx), C.byref(prob), float(rho), C.byref(opt)))
        self._ctx = ctx
        self.n, self.p, self.rho = n, p, float(rho)
        self.format = fmt
        self.world_size, self.rank = o["world_size"], o["rank"]
        self.batch = batch
        if batch > 1:     # whole QPs are sharded, not rows
            self.b_range = shard_range(batch, self.world_size, self.rank)
            self.n_range, self.p_range = (0, n), (0, p)
        else:
            self.b_range = (0, 1)
            r0, nl, s0, pl = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()   # the context's row ranges
            L.check(lib.duquad_local_ranges(ctx, C.byref(r0), C.byref(nl), C.byref(s0), C.byref(pl)), ctx)
            self.n_range = (r0.value, r0.value + nl.value)
            self.p_range = (s0.value, s0.value + pl.value)
        self.device = o["device"]
        self.last_result = None

    # ------------------------------------------------------------------ API
    def lipschitz(self, iters: int = 100, safety: float = 1e-6):
        """duquad_lipschitz: (L_in, L_d, ||G||^2).  `safety` inflates both eigen estimates (Lanczos
        Ritz values never exceed the true eigenvalues, so L_in and L_d must be over-estimates;
        SPEC.md:76's delta_safe = 1e-6); the returned ||G||^2 is the raw estimate."""
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        L.check(self._lib.duquad_lipschitz(self._ctx, iters, safety, C.byref(a), C.byref(b), C.byref(c)),
                self._ctx)
        return a.value, b.value, c.value

    def set_constants(self, L_in: float, L_d: float):
        L.check(self._lib.duquad_set_constants(self._ctx, float(L_in), float(L_d)), self._ctx)

    def set_trace(self, lam_trace=None, u_trace=None, max_outer: int = 0):
        """Device (torch CUDA) buffers of shape (max_outer, p_local) / (max_outer, n_local)."""
        self._trace = (lam_trace, u_trace)
        L.check(self._lib.duquad_set_trace(self._ctx, lam_trace.data_ptr() if lam_trace is not None else None,
                                           u_trace.data_ptr() if u_trace is not None else None,
                                           int(max_outer)), self._ctx)

    def solve(self, alg: str = "DFGM", outer: int = 1, inner: int = 1) -> dict:
        res = L.Result()
        L.check(self._lib.duquad_solve(self._ctx, _ALGS[alg], int(outer), int(inner), C.byref(res)), self._ctx)
        self.last_result = {k: getattr(res, k) for k, _ in L.Result._fields_}
        return self.last_result

    def set_initial(self, x0=None, lambda0=None):
        """Warm start for subsequent solves (duquad_set_initial): u_bar^0 = [x0]_U, lambda^0 = lambda0.
        Full vectors (batch: (B, n) / (B, p)), NumPy or torch (host or CUDA); None resets."""
        xs = _Arr(x0, np.float64) if x0 is not None else None
        ls = _Arr(lambda0, np.float64) if lambda0 is not None else None
        dev = bool((xs and xs.dev) or (ls and ls.dev))
        if xs and ls and xs.dev != ls.dev:
            raise ValueError("x0 and lambda0 must both be host or both be device arrays")
        L.check(self._lib.duquad_set_initial(self._ctx, xs.ptr if xs else None, ls.ptr if ls else None, int(dev)),
                self._ctx)
        self._init_keep = (xs, ls)

    def solve_eps(self, alg: str = "DFGM", outer: int = 1, inner_max: int = 1000, eps_in: float = 1e-6,
                  sigma_L: float = 1.0) -> dict:
        """DFOM with eps_in-driven inner stopping (duquad_solve_eps).  The report gets 'inner_counts'
        and 'converged' (per outer iteration + the last-iterate solve) and 'capped' (EMAXITER)."""
        res = L.Result()
        st = self._lib.duquad_solve_eps(self._ctx, _ALGS[alg], int(outer), int(inner_max), float(eps_in),
                                        float(sigma_L), C.byref(res))
        if st not in (L.DUQUAD_OK, L.DUQUAD_EMAXITER):
            L.check(st, self._ctx)
        info = {k: getattr(res, k) for k, _ in L.Result._fields_}
        bl = self.b_range[1] - self.b_range[0] if self.batch > 1 else 1
        m = (int(outer) + 1) * bl
        counts = (C.c_int32 * m)()
        conv = (C.c_int32 * m)()
        L.check(self._lib.duquad_get_inner_counts(self._ctx, counts, conv, m), self._ctx)
        info["inner_counts"] = list(counts)
        info["converged"] = [bool(c) for c in conv]
        if self.batch > 1:   # per QP: [QP][solve]
            k1 = int(outer) + 1
            info["inner_counts"] = [info["inner_counts"][b * k1:(b + 1) * k1] for b in range(bl)]
            info["converged"] = [info["converged"][b * k1:(b + 1) * k1] for b in range(bl)]
        info["capped"] = st == L.DUQUAD_EMAXITER
        self.last_result = info
        return info

    def result(self, device: bool = False):
        """(x_last, x_avg, lambda) local slices; NumPy on the host or torch on the device.
        Batched: arrays of shape (B_local, n) / (B_local, p)."""
        nl = self.n_range[1] - self.n_range[0]
        pl = self.p_range[1] - self.p_range[0]
        bl = self.b_range[1] - self.b_range[0]
        shp_n = (bl, nl) if self.batch > 1 else (nl,)
        shp_p = (bl, max(pl, 1)) if self.batch > 1 else (max(pl, 1),)
        if device:
            import torch
            dev = torch.device("cuda", torch.cuda.current_device() if self.device < 0 else self.device)
            xl = torch.empty(shp_n, dtype=torch.float64, device=dev)
            xa = torch.empty(shp_n, dtype=torch.float64, device=dev)
            lam = torch.empty(shp_p, dtype=torch.float64, device=dev)
            L.check(self._lib.duquad_get_result(self._ctx, xl.data_ptr(), xa.data_ptr(), lam.data_ptr(), 1),
                    self._ctx)
            return xl, xa, lam[..., :pl]
        xl = np.empty(shp_n)
        xa = np.empty(shp_n)
        lam = np.empty(shp_p)
        L.check(self._lib.duquad_get_result(self._ctx, xl.ctypes.data, xa.ctypes.data, lam.ctypes.data, 0),
                self._ctx)
        return xl, xa, lam[..., :pl]

    def get_state(self) -> dict:
        """The DFOM state the last solve snapshotted after its K-th outer iteration (needs
        checkpoint=True): x = u_bar^K, mu = mu^K, lam_prev = lambda^{K-1}, x_avg, outer_done, S."""
        bl = self.b_range[1] - self.b_range[0]
        nl = self.n_range[1] - self.n_range[0]     # row-sharded: this rank's slices
        pl = self.p_range[1] - self.p_range[0]
        shp_n = (bl, nl) if self.batch > 1 else (nl,)
        shp_p = (bl, max(pl, 1)) if self.batch > 1 else (max(pl, 1),)
        x, xa = np.empty(shp_n), np.empty(shp_n)
        mu, lp = np.empty(shp_p), np.empty(shp_p)
        j, S = C.c_int64(), C.c_double()
        L.check(self._lib.duquad_get_state(self._ctx, x.ctypes.data, mu.ctypes.data, lp.ctypes.data, xa.ctypes.data,
                                           C.byref(j), C.byref(S), 0), self._ctx)
        return dict(x=x, mu=mu[..., :pl], lam_prev=lp[..., :pl], x_avg=xa, outer_done=j.value, S=S.value)

    def set_state(self, state: dict):
        """Continue the next solve from `state` (a get_state() dict): outer iterations
        outer_done + 1, ...; solve(K1), get_state, set_state, solve(K2) == solve(K1 + K2)."""
        arrs = [_Arr(np.ascontiguousarray(state[k], np.float64), np.float64) for k in ("x", "mu", "lam_prev", "x_avg")]
        L.check(self._lib.duquad_set_state(self._ctx, arrs[0].ptr, arrs[1].ptr, arrs[2].ptr, arrs[3].ptr,
                                           int(state["outer_done"]), float(state["S"]), 0), self._ctx)

    TRACE_FIELDS = ("k", "dual_val", "f_last", "f_avg", "infeas_last", "infeas_avg", "inner_iters", "cum_matvecs")

    def solve_monitored(self, alg: str = "DFGM", outer_max: int = 1, inner: int = 1, check_every: int = 1,
                        which: str = "avg", eps: float = 1e-2, F_star: float = float("nan")) -> dict:
        """DFOM with the stopping test checked every check_every outer iterations
        (duquad_solve_monitored): stop at the first checked j with dist_K <= eps and
        |F - F_star| <= eps, or (F_star NaN) |F - d_bar(lambda^j)| <= eps (1 + |F|).  The report
        adds the duquad_monitor fields and 'history' (one dict per check, TRACE_FIELDS);
        result() is bitwise solve(alg, outer_done, inner)'s."""
        res, mon = L.Result(), L.Monitor()
        cap = -(-int(outer_max) // max(int(check_every), 1))
        hist = (C.c_double * (8 * max(cap, 1)))()
        L.check(self._lib.duquad_solve_monitored(self._ctx, _ALGS[alg], int(outer_max), int(inner), int(check_every),
                                                 0 if which == "last" else 1, float(eps), float(F_star),
                                                 C.byref(mon), hist, C.byref(res)), self._ctx)
        info = {k: getattr(res, k) for k, _ in L.Result._fields_}
        info.update({k: getattr(mon, k) for k, _ in L.Monitor._fields_})
        info["converged"] = bool(info["converged"])
        h = np.frombuffer(hist, dtype=np.float64).reshape(-1, 8)[:info["checks"]]
        info["history"] = [dict(zip(self.TRACE_FIELDS, (int(r[0]), *map(float, r[1:6]), int(r[6]), int(r[7]))))
                           for r in h]
        self.last_result = info
        return info

    @classmethod
    def write_trace_csv(cls, path, history):
        """The per-check history of solve_monitored as CSV (SPEC trace export header)."""
        with open(path, "w") as f:
            f.write(",".join(cls.TRACE_FIELDS) + "\n")
            for r in history:
                f.write(",".join(repr(r[k]) for k in cls.TRACE_FIELDS) + "\n")

    def residuals(self, which: str = "last"):
        F, d, lag = C.c_double(), C.c_double(), C.c_double()
        L.check(self._lib.duquad_residuals(self._ctx, 0 if which == "last" else 1, C.byref(F), C.byref(d),
                                           C.byref(lag)), self._ctx)
        return F.value, d.value, lag.value

    def close(self):
        if getattr(self, "_ctx", None):
            self._lib.duquad_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
