"""CPU oracle for DuQuad's DGM / DFGM (arXiv 1504.05708) -- TEST INFRASTRUCTURE.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this module.  The product path
(`paper_1504_05708_b200/`) never imports, links or executes it, and this
module imports nothing from the product path.

A plain, slow, obviously-correct fp64 NumPy replay of the paper's
algorithms, step by step, in the paper's order and notation.  Citations are
PAPER.md line numbers ("P:n") plus the equation / algorithm label.
Library primitives used as single steps: `@` (matrix-vector / matrix-matrix
product; dense ndarray or scipy.sparse), np.sqrt, np.minimum / np.maximum.

Readings of passages where the paper is silent or ambiguous are the ones of
SURVEY.md §8(c) and are listed in DESIGN.md §2 (c1..c20); each is marked
"[reading cN]" below.

Shapes: `u` may be a vector (n,) or a matrix (n, B) whose columns are B
independent QPs sharing Q and G (config 3); then q is (n, B), g is (p, B)
and every multiplier is (p, B).  Every operation below is column-wise.

Parity: pinned by tests/test_oracle_pins.py (closed forms, SPEC worked
examples, brute-force active-set enumeration, KKT solves, theta identities,
weak duality, Theorem 1 / Lemma 1 envelopes).  No function here is
"parity unpinned".
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

ZERO = 0      # row of K = {0}     (equality)
NONPOS = 1    # row of K = R^p_-   (inequality)

DGM = "DGM"
DFGM = "DFGM"

INNER_FGM = "FGM"
INNER_GM = "GM"
INNER_FGM_SIGMA = "FGM_SIGMA"


# ---------------------------------------------------------------- sequences
def theta_sequence(k_max: int) -> np.ndarray:
    """theta_1..theta_{k_max}: theta_1 = 1, theta_{k+1} = (1 + sqrt(1 + 4 theta_k^2)) / 2.

    P:358-363 (FGM rule) and P:587-589 (DFGM rule).  Returned array is
    1-based: out[k] = theta_k, out[0] unused (= 0).
    """
    th = np.zeros(k_max + 1)
    if k_max >= 1:
        th[1] = 1.0
    for k in range(1, k_max):
        th[k + 1] = (1.0 + np.sqrt(1.0 + 4.0 * th[k] * th[k])) / 2.0
    return th


def beta_fgm(k_max: int) -> np.ndarray:
    """beta_k = (theta_k - 1) / theta_{k+1}, k = 1..k_max.  1-based."""
    th = theta_sequence(k_max + 1)
    b = np.zeros(k_max + 1)
    for k in range(1, k_max + 1):
        b[k] = (th[k] - 1.0) / th[k + 1]
    return b


def beta_fgm_sigma(L: float, sigma: float) -> float:
    """FGM_sigma: beta = (sqrt(L) - sqrt(sigma)) / (sqrt(L) + sqrt(sigma))."""
    return (np.sqrt(L) - np.sqrt(sigma)) / (np.sqrt(L) + np.sqrt(sigma))


# -------------------------------------------------------------- projections
def _cone_col(cone, v):
    c = np.asarray(cone)
    return c if v.ndim == 1 else c[:, None]


def proj_K(v: np.ndarray, cone: np.ndarray) -> np.ndarray:
    """[v]_K: ZERO rows -> 0, NONPOS rows -> min(v, 0).  K of P:201-202; notation P:170-180."""
    c = _cone_col(cone, v)
    return np.where(c == NONPOS, np.minimum(v, 0.0), 0.0)


def dist_K(v: np.ndarray, cone: np.ndarray):
    """dist_K(v) = ||v - [v]_K|| (per column for a batch).  Notation P:170-180."""
    d = v - proj_K(v, cone)
    return np.sqrt(np.sum(d * d, axis=0))


def proj_Kd(v: np.ndarray, cone: np.ndarray, project_dual: bool) -> np.ndarray:
    """[v]_{K_d}.  K_d = R^p_+ if Q > 0 and K = R^p_- , else R^p.

    [reading c3] with project_dual the NONPOS rows are projected onto R_+
    (the literal Q > 0 rule, and the north_star's "projected onto K*");
    ZERO rows are never projected (their dual set is R).
    """
    if not project_dual:
        return v.copy()
    c = _cone_col(cone, v)
    return np.where(c == NONPOS, np.maximum(v, 0.0), v)


def clamp_U(v: np.ndarray, lb: np.ndarray, ub: np.ndarray) -> np.ndarray:
    """[v]_U for the box U = [lb, ub]."""
    if v.ndim == 2:
        lb = lb[:, None]
        ub = ub[:, None]
    return np.minimum(np.maximum(v, lb), ub)


# ------------------------------------------------------- (augmented) Lagrangian
def objective(Q, q, u):
    """F(u) = 1/2 u'Qu + q'u (Eq. original_primal); per column for a batch."""
    Qu = Q @ u
    return 0.5 * np.sum(u * Qu, axis=0) + np.sum(q * u, axis=0)


def slack(r: np.ndarray, lam: np.ndarray, cone, rho: float) -> np.ndarray:
    """s(u, lambda) with r = Gu + g:
    [r + lambda/rho]_K if rho > 0, 0 if rho = 0."""
    if rho > 0:
        return proj_K(r + lam / rho, cone)
    return np.zeros_like(r)


def aug_lagrangian(Q, q, G, g, cone, rho, u, lam):
    """L_rho(u, lambda) in the closed form (auglag1)."""
    r = G @ u + g
    if rho > 0:
        d = dist_K(r + lam / rho, cone)
        return objective(Q, q, u) + 0.5 * rho * d * d - np.sum(lam * lam, axis=0) / (2.0 * rho)
    return objective(Q, q, u) + np.sum(lam * r, axis=0)


def aug_lagrangian_grad(Q, q, G, g, cone, rho, u, lam):
    """grad_u L_rho(u, lambda), differentiating (auglag1):

    rho > 0: Qu + q + rho G'(w - [w]_K), w = Gu + g + lambda/rho
             (grad of dist_K(w)^2 / 2 is w - [w]_K);
    rho = 0: Qu + q + G'lambda.
    For K = {0} this equals the paper's (Q + rho G'G)u + (q + G'mu + rho G'g),
    P:1266-1267 (pinned in tests).
    """
    if rho > 0:
        w = G @ u + g + lam / rho
        v = rho * (w - proj_K(w, cone))
    else:
        v = lam
    return Q @ u + q + G.T @ v


# ------------------------------------------------------------- Algorithm FOM
def fom(grad_fn, x0, L, lb, ub, iters: int, rule: str = INNER_FGM, sigma: float = 0.0,
        history: Optional[list] = None):
    """Algorithm FOM(phi, X), with X = the box U.

    Given x^0 = y^1 in X, for k >= 1:
        x^k     = [y^k - grad phi(y^k) / L]_X
        y^{k+1} = x^k + beta_k (x^k - x^{k-1})
    beta rule: GM beta = 0; FGM theta recurrence;
    FGM_sigma constant beta.  [reading c5] theta restarts at
    theta_1 = 1 on every call.  [reading c6] returns x^{iters} (not y).
    """
    x, _, _ = fom_run(grad_fn, x0, L, lb, ub, iters, rule, sigma, history=history)
    return x


def fom_run(grad_fn, x0, L, lb, ub, iters: int, rule: str = INNER_FGM, sigma: float = 0.0,
            eps_in: Optional[float] = None, sigma_L: Optional[float] = None,
            history: Optional[list] = None, gm: Optional[list] = None):
    """Algorithm FOM as in fom(), optionally stopped by the inner accuracy eps_in.

    Stopping test (reading c15 of Eq. duquad_in): after step k,
    stop with u_bar = x^k when the gradient map at y^k satisfies
        L * ||y^k - x^k|| <= sqrt(2 * sigma_L * eps_in),
    which for a sigma_L-strongly convex phi gives phi(x^k) - phi* <= eps_in
    (phi(x+) - phi* <= ||G_L(y)||^2 / (2 sigma_L) for the gradient map G_L(y) = L (y - x+)).
    `iters` is then the cap.  Returns (x, steps run, converged).  `gm` collects
    L * ||y^k - x^k|| per step.
    """
    if rule == INNER_FGM:
        beta = beta_fgm(iters)
    elif rule == INNER_GM:
        beta = np.zeros(iters + 1)
    elif rule == INNER_FGM_SIGMA:
        beta = np.full(iters + 1, beta_fgm_sigma(L, sigma))
    else:
        raise ValueError(rule)
    thr = None if eps_in is None else np.sqrt(2.0 * sigma_L * eps_in)
    x_prev = x0.copy()
    y = x0.copy()
    for k in range(1, iters + 1):
        x = clamp_U(y - grad_fn(y) / L, lb, ub)
        if history is not None:
            history.append(x.copy())
        if thr is not None or gm is not None:
            g_k = L * float(np.linalg.norm(y - x))
            if gm is not None:
                gm.append(g_k)
            if thr is not None and g_k <= thr:
                return x, k, True
        y = x + beta[k] * (x - x_prev)
        x_prev = x
    return x_prev, iters, thr is None


def inner_solve(Q, q, G, g, cone, rho, mu, x0, L_in, lb, ub, iters,
                rule=INNER_FGM, sigma=0.0, eps_in=None, sigma_L=None, gm=None, info=None):
    """Step 1 of DuQuad: u_bar(mu) by FOM(L_rho(., mu), U) warm-started at x0
    (P:601-603); fixed `iters` steps, or stopped by the inner accuracy eps_in (fom_run).
    `info`, if a list, receives (steps run, converged)."""
    def grad(u):
        return aug_lagrangian_grad(Q, q, G, g, cone, rho, u, mu)
    x, k, conv = fom_run(grad, x0, L_in, lb, ub, iters, rule, sigma, eps_in, sigma_L, gm=gm)
    if info is not None:
        info.append((k, conv))
    return x


def inexact_dual_grad(G, g, cone, rho, u_bar, mu):
    """grad_bar d_rho(mu) = G u_bar + g - s(u_bar, mu), Eq. (inexact_framework) P:490-493."""
    r = G @ u_bar + g
    return r - slack(r, mu, cone, rho)


# ------------------------------------------------------------ Algorithm DFOM
@dataclass
class DfomResult:
    x_last: np.ndarray          # u_bar(lambda^K), Eq. (last_primal)
    x_avg: np.ndarray           # Eq. (average_primal)
    lam: np.ndarray             # lambda^K
    u_bar_K: np.ndarray         # u_bar^K = u_bar(mu^K)
    S: float                    # S_K = sum of weights
    trace_lam: List[np.ndarray] = field(default_factory=list)   # lambda^j, j=1..K
    trace_u: List[np.ndarray] = field(default_factory=list)     # u_bar^j, j=1..K
    trace_mu: List[np.ndarray] = field(default_factory=list)    # mu^j, j=1..K
    inner_counts: List[int] = field(default_factory=list)       # steps per inner solve (K + 1)
    converged: List[bool] = field(default_factory=list)         # eps_in test met (eps mode)
    gm: List[List[float]] = field(default_factory=list)         # L ||y^k - x^k|| per step (record_gm)
    lam_hat: Optional[np.ndarray] = None                          # dual average (dual_average=True)


def dfom(Q, q, G, g, lb, ub, cone, rho: float, alg: str, outer: int, inner,
         L_in: float, L_d: float, inner_rule: str = INNER_FGM, sigma: float = 0.0,
         dual_step_scale: float = 0.5, project_dual: bool = True,
         lam0: Optional[np.ndarray] = None, keep_trace: bool = False,
         eps_in: Optional[float] = None, sigma_L: Optional[float] = None,
         record_gm: bool = False, x0: Optional[np.ndarray] = None,
         dual_average: bool = False) -> DfomResult:
    """Algorithm DFOM(d_rho, K_d), with fixed inner iteration counts.

    Given lambda^0 = mu^1 in K_d (= 0, [reading c8]), for k >= 1:
      1. u_bar^k = u_bar(mu^k), FOM warm-started at u_bar^{k-1}
      2. lambda^k = [mu^k + grad_bar d(mu^k) / (2 L_d)]_{K_d} [reading c1]
      3. mu^{k+1} = lambda^k + beta_k (lambda^k - lambda^{k-1})
    beta_k = 0 for DGM; theta recurrence for DFGM.
    u_bar^0 = [0]_U [reading c7].
    Primal average: sum_j theta_j u_bar^j / S_k, theta_j = 1 for DGM
      (Eq. average_primal) [reading c9].
    Last iterate: u_bar(lambda^K) by one more inner solve warm-started at
      u_bar^K (Eq. last_primal) [reading c10].
    dual_step_scale = 1/2 gives the paper's 1/(2 L_d); project_dual per [reading c3].
    `inner`: steps per inner solve (int), or a sequence of K + 1 per-solve counts (the last
    for the last-iterate solve); with eps_in and sigma_L the inner solves stop by the
    eps_in test of fom_run (NEXT-1) and `inner` is the cap.
    Warm start (NEXT-2): x0 gives u_bar^0 = [x0]_U, lam0 gives lambda^0 = mu^1 (must lie in K_d).
    DGM dual averaging (NEXT-2): with dual_average=True (DGM only) the returned dual
    point is lambda^K := [lam_hat + grad_bar d(lam_hat) / (2 L_d)]_{K_d} with the average
    lam_hat = (1 / (K+1)) sum_{j=0}^{K} lambda^j, grad_bar d(lam_hat) from one more inner solve
    at mu = lam_hat (warm-started at u_bar^K), and the last iterate is u_bar of that point
    (warm-started at u_bar(lam_hat)); K + 2 inner solves in all.
    """
    nsolve = outer + (2 if dual_average else 1)
    if dual_average and alg != DGM:
        raise ValueError("dual averaging is the DGM final-point rule (P:624-626)")
    counts = [int(inner)] * nsolve if np.ndim(inner) == 0 else [int(c) for c in inner]
    if outer < 1 or len(counts) != nsolve or min(counts) < 1:
        raise ValueError("outer >= 1 and inner >= 1 (one count per solve: K + 1, K + 2 with dual_average)")
    p = G.shape[0]
    bshape = (p,) if q.ndim == 1 else (p, q.shape[1])
    theta = theta_sequence(outer + 1)
    lam_prev = np.zeros(bshape) if lam0 is None else lam0.copy()   # lambda^0
    mu = lam_prev.copy()                                            # mu^1 = lambda^0
    u_bar = clamp_U(np.zeros(q.shape) if x0 is None else np.asarray(x0, float), lb, ub)   # u_bar^0
    xsum = np.zeros(q.shape)
    S = 0.0
    lam_sum = lam_prev.copy()                                       # sum_{j=0}^{k} lambda^j
    res = DfomResult(None, None, None, None, 0.0)
    info = []

    def gm_list():
        if not record_gm:
            return None
        res.gm.append([])
        return res.gm[-1]

    for k in range(1, outer + 1):
        u_bar = inner_solve(Q, q, G, g, cone, rho, mu, u_bar, L_in, lb, ub, counts[k - 1],
                            inner_rule, sigma, eps_in, sigma_L, gm_list(), info)    # step 1
        gbar = inexact_dual_grad(G, g, cone, rho, u_bar, mu)
        lam = proj_Kd(mu + (dual_step_scale / L_d) * gbar, cone, project_dual)     # step 2
        omega = theta[k] if alg == DFGM else 1.0
        xsum = xsum + omega * u_bar
        S = S + omega
        if alg == DFGM:
            beta_k = (theta[k] - 1.0) / theta[k + 1]
        elif alg == DGM:
            beta_k = 0.0
        else:
            raise ValueError(alg)
        if keep_trace:
            res.trace_mu.append(mu.copy())
            res.trace_lam.append(lam.copy())
            res.trace_u.append(u_bar.copy())
        mu = lam + beta_k * (lam - lam_prev)                                       # step 3
        lam_prev = lam
        lam_sum = lam_sum + lam
    if dual_average:   # the final dual point from the average of lambda^0..lambda^K
        lam_hat = lam_sum / (outer + 1)
        u_hat = inner_solve(Q, q, G, g, cone, rho, lam_hat, u_bar, L_in, lb, ub, counts[outer],
                            inner_rule, sigma, eps_in, sigma_L, gm_list(), info)
        lam_prev = proj_Kd(lam_hat + (dual_step_scale / L_d) * inexact_dual_grad(G, g, cone, rho, u_hat, lam_hat),
                           cone, project_dual)
        res.lam_hat = lam_hat
        u_bar_last, c_last = u_hat, counts[outer + 1]
    else:
        u_bar_last, c_last = u_bar, counts[outer]
    x_last = inner_solve(Q, q, G, g, cone, rho, lam_prev, u_bar_last, L_in, lb, ub, c_last,
                         inner_rule, sigma, eps_in, sigma_L, gm_list(), info)
    res.inner_counts = [c for c, _ in info]
    res.converged = [v for _, v in info]
    res.x_last = x_last
    res.x_avg = xsum / S
    res.lam = lam_prev
    res.u_bar_K = u_bar
    res.S = S
    return res


# ------------------------------------------------------------ theory schedule (NEXT-1)
def theory_schedule(alg: str, eps: float, R_d: float, L_d: float, L_in: float, sigma_L: float,
                    D_U: float, normG: float, lambda_min_Q: float = 0.0, lambda_max_Q: float = 0.0) -> dict:
    """DuQuad's parameter choices for a target accuracy eps.

    eps_in, k_out: Eq. (choose_ein), P:641-652 (each term of Theorem 1's bound
      (bound_gen_dfg), at most eps/2), counts rounded up.
    k_in: proof of Theorem in:th_last, P:1168-1173 (Lemma 1 (bound_gen_dfg1), P:386-391,
      with R_phi <= D_U), rounded up.
    rho_star = 8 R_d^2 / eps.
    k_total: Theorem in:th_last, P:1162-1169 (floor, as printed); the log's argument is taken as
      at least 1 (||G|| = 0 couples nothing: 0 outer work, not 0 * log 0).
    case: P:252-258, 1 if Q > 0 (rho = 0), else 2 (rho > 0); "Q > 0" numerically as
      lambda_min(Q) > tau_pd = 1e-7 max(1, lambda_max(Q)) (reading c25).
    """
    q8 = 8.0 * L_d * R_d ** 2 / eps
    if alg == DGM:
        eps_in, k_out = eps / 4.0, int(np.ceil(q8))
    elif alg == DFGM:
        eps_in, k_out = eps * np.sqrt(eps) / (8.0 * R_d * np.sqrt(2.0 * L_d)), int(np.ceil(np.sqrt(q8)))
    else:
        raise ValueError(alg)
    if sigma_L > 0:
        k_in = np.sqrt(L_in / sigma_L) * np.log(L_in * D_U ** 2 / eps_in) + 1.0
        k_total = 16.0 * normG * R_d / np.sqrt(sigma_L * eps) * np.log(max(1.0, 8.0 * normG * D_U * R_d / eps))
    else:
        k_in = np.sqrt(2.0 * L_in * D_U ** 2 / eps_in)
        k_total = 24.0 * normG * D_U * R_d / eps
    return dict(eps_in=float(eps_in), k_out=k_out, k_in=int(np.ceil(max(k_in, 1.0))),
                rho_star=8.0 * R_d ** 2 / eps, k_total=int(np.floor(k_total)),
                case_id=1 if lambda_min_Q > 1e-7 * max(1.0, lambda_max_Q) else 2)


def theorem1_bound(alg: str, k: int, L_d: float, R_d: float, eps_in: float) -> float:
    """Right-hand side of Theorem 1 (bound_gen_dfg), P:614-616:
    4 L_d R_d^2 / (k+1)^p + 2 (k+1)^(p-1) eps_in, p = 1 (DGM) or 2 (DFGM) (Eq. pbetak)."""
    p = 1 if alg == DGM else 2
    return 4.0 * L_d * R_d ** 2 / (k + 1) ** p + 2.0 * (k + 1) ** (p - 1) * eps_in


def drift_bound(k: int, L_d: float, R_d: float, eps_in: float) -> float:
    """Multiplier drift (bound_seq_dgm): ||lambda^k - lambda*|| <= R_d + sqrt(k eps_in / L_d)."""
    return R_d + np.sqrt(k * eps_in / L_d)


def feas_last_bound(alg: str, k: int, L_d: float, R_d: float, eps_in: float) -> float:
    """Infeasibility of the last primal iterate u_bar(lambda^k), (aux_feas_bound) P:805-810:
    d_K(G u_bar + g) <= sqrt(2 L_d eps_in) + sqrt(2 L_d (F* - d(lambda^k))), the dual gap bounded by
    Theorem 1."""
    return np.sqrt(2.0 * L_d * eps_in) + np.sqrt(2.0 * L_d * theorem1_bound(alg, k, L_d, R_d, eps_in))


def feas_avg_bound(alg: str, K: int, L_d: float, R_d: float, eps_in: float) -> float:
    """Infeasibility of the primal average over K outer iterates:
    DGM (feasibility_final): (2 L_d / K) ||lambda^K - lambda^0|| <= 4 L_d R_d / K + 2 sqrt(L_d eps_in / K);
    DFGM (infes_av): 8 L_d R_d / K^2 + 8 sqrt(L_d eps_in / K)  (the paper's k+1 = K terms)."""
    if alg == DGM:
        return 4.0 * L_d * R_d / K + 2.0 * np.sqrt(L_d * eps_in / K)
    return 8.0 * L_d * R_d / K ** 2 + 8.0 * np.sqrt(L_d * eps_in / K)


def lemma1_bound(k: int, L: float, sigma: float, R: float, p: int = 2) -> float:
    """Right-hand side of Lemma 1 (bound_gen_dfg1)."""
    lin = (1.0 - np.sqrt(sigma / L)) ** (k - 1) * L * R ** 2 if sigma > 0 else np.inf
    return min(lin, 2.0 * L * R ** 2 / (k + 1) ** p)


# ------------------------------------------------------------ constants / checks
def lipschitz_constants(Q, G, rho: float, lambda_min_lb: float, l_mode: int = 0,
                        safety: float = 0.0):
    """L_in and L_d from their definitions, by symmetric eigen-decomposition.

    l_mode 0: L_in = lambda_max(Q + rho G'G)  (north_star; Hessian of L_rho for K={0})
    l_mode 1: L_in = lambda_max(Q) + rho ||G||^2
    L_d = ||G||^2 / (lambda_min(Q) + rho ||G||^2), Eq. (Ld), with a caller
    lower bound in place of lambda_min(Q) [reading c13].
    Returns (L_in, L_d, ||G||^2).  Dense inputs only.
    """
    GtG = G.T @ G
    normG2 = float(np.linalg.eigvalsh(GtG)[-1]) if G.shape[0] > 0 else 0.0
    if l_mode == 0:
        lmax = float(np.linalg.eigvalsh(Q + rho * GtG)[-1])
    else:
        lmax = float(np.linalg.eigvalsh(Q)[-1]) + rho * normG2
    L_in = (1.0 + safety) * lmax
    # safety inflates every eigen-derived constant (SPEC.md:76 delta_safe): L_d is increasing
    # in ||G||^2, so it is formed from the inflated value; the raw ||G||^2 is returned
    nG2_up = (1.0 + safety) * normG2
    denom = lambda_min_lb + rho * nG2_up
    L_d = nG2_up / denom if denom > 0 else float("inf")
    return L_in, L_d, normG2


def dual_value(Q, q, G, g, lb, ub, cone, rho, lam, L_in, inner_iters=20000, x0=None):
    """d_rho(lambda) = min_{u in U} L_rho(u, lambda) (Eq. dual_fc), evaluated
    as L_rho(u_bar, lambda) after a long FOM run.  Returns (value, u_bar)."""
    n = Q.shape[0]
    if x0 is None:
        x0 = clamp_U(np.zeros(q.shape), lb, ub)
    u = inner_solve(Q, q, G, g, cone, rho, lam, x0, L_in, lb, ub, inner_iters)
    return aug_lagrangian(Q, q, G, g, cone, rho, u, lam), u
