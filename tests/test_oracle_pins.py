"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test cites the passage whose value / closed form / invariant it uses:
P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.  Golden
values live in tests/golden/spec_examples.json with their citations.
"""
import math

import numpy as np
import pytest

import qpgen
from oracle import dfom as O
from oracle import kkt


def _a(x):
    return np.asarray(x, dtype=float)


# ------------------------------------------------------------------ geometry
def test_proj_dist_slack_examples(golden):
    for ex in golden["proj_K"]:
        assert np.array_equal(O.proj_K(_a(ex["v"]), np.array(ex["cone"])), _a(ex["out"])), ex["cite"]
    for ex in golden["dist_K"]:
        assert O.dist_K(_a(ex["v"]), np.array(ex["cone"])) == pytest.approx(ex["out"]), ex["cite"]
    for ex in golden["slack"]:
        out = O.slack(_a(ex["r"]), _a(ex["lam"]), np.array(ex["cone"]), ex["rho"])
        assert np.array_equal(out, _a(ex["out"])), ex["cite"]


def test_lagrangian_value_examples(golden):
    for ex in golden["lagrangian_value"]:
        v = O.aug_lagrangian(_a(ex["Q"]), _a(ex["q"]), _a(ex["G"]), _a(ex["g"]),
                             np.array(ex["cone"]), ex["rho"], _a(ex["u"]), _a(ex["lam"]))
        assert v == pytest.approx(ex["out"], abs=1e-14), ex["cite"]


def test_lagrangian_grad_examples(golden):
    for ex in golden["lagrangian_grad"]:
        v = O.aug_lagrangian_grad(_a(ex["Q"]), _a(ex["q"]), _a(ex["G"]), _a(ex["g"]),
                                  np.array(ex["cone"]), ex["rho"], _a(ex["u"]), _a(ex["lam"]))
        assert np.allclose(v, _a(ex["out"]), atol=1e-14), ex["cite"]


def test_closed_form_matches_min_over_slack():
    """(auglag1) P:243-251 vs the definition (auglag), min over s in K done
    numerically per row with a bounded scalar minimiser (independent path)."""
    from scipy.optimize import minimize_scalar
    prob = qpgen.tiny(4, 5, seed=3, kind="mixed")
    rng = np.random.default_rng(11)
    for rho in (0.5, 2.0):
        u = rng.uniform(-1, 1, prob.n)
        lam = rng.normal(size=prob.p)
        r = prob.G @ u + prob.g
        val = 0.5 * u @ prob.Q @ u + prob.q @ u
        for i in range(prob.p):
            f = lambda s: lam[i] * (r[i] - s) + 0.5 * rho * (r[i] - s) ** 2
            if prob.cone[i] == qpgen.ZERO:
                val += f(0.0)
            else:
                m = minimize_scalar(f, bounds=(-50.0, 0.0), method="bounded",
                                    options=dict(xatol=1e-12))
                val += min(m.fun, f(0.0))
        cf = O.aug_lagrangian(prob.Q, prob.q, prob.G, prob.g, prob.cone, rho, u, lam)
        assert cf == pytest.approx(val, rel=1e-9, abs=1e-9)


def test_grad_matches_finite_differences():
    """gradient vs central differences of the value."""
    prob = qpgen.tiny(6, 5, seed=5, kind="mixed")
    rng = np.random.default_rng(7)
    for rho in (0.0, 1.0, 3.0):
        for _ in range(10):
            u = rng.uniform(-1, 1, prob.n)
            lam = rng.normal(size=prob.p)
            gr = O.aug_lagrangian_grad(prob.Q, prob.q, prob.G, prob.g, prob.cone, rho, u, lam)
            h = 1e-6
            fd = np.zeros(prob.n)
            for j in range(prob.n):
                e = np.zeros(prob.n)
                e[j] = h
                fd[j] = (O.aug_lagrangian(prob.Q, prob.q, prob.G, prob.g, prob.cone, rho, u + e, lam)
                         - O.aug_lagrangian(prob.Q, prob.q, prob.G, prob.g, prob.cone, rho, u - e, lam)) / (2 * h)
            assert np.allclose(gr, fd, rtol=1e-5, atol=1e-6)


def test_grad_equality_closed_form():
    """for K = {0}, grad = (Q + rho G'G)u + (q + G'mu + rho G'g)."""
    prob = qpgen.tiny(7, 4, seed=9, kind="eq")
    rng = np.random.default_rng(2)
    u = rng.uniform(-1, 1, prob.n)
    mu = rng.normal(size=prob.p)
    for rho in (0.0, 0.7, 5.0):
        H = prob.Q + rho * prob.G.T @ prob.G
        ref = H @ u + (prob.q + prob.G.T @ mu + rho * prob.G.T @ prob.g)
        got = O.aug_lagrangian_grad(prob.Q, prob.q, prob.G, prob.g, prob.cone, rho, u, mu)
        assert np.allclose(got, ref, rtol=1e-12, atol=1e-12)


# ----------------------------------------------------------------- sequences
def test_theta_identities(golden):
    th = O.theta_sequence(10001)
    assert th[1] == 1.0
    assert th[2] == pytest.approx((1 + math.sqrt(5)) / 2, rel=1e-15)
    assert th[3] == pytest.approx(golden["theta"]["theta3_approx"], abs=1e-5)
    S = np.cumsum(th[1:])                                                       # S_k, j=1..k
    k = np.arange(1, 10002)
    assert np.all((k + 1) / 2 <= th[1:] + 1e-12) and np.all(th[1:] <= k + 1e-12)
    assert np.allclose(S, th[1:] ** 2, rtol=1e-9)
    b = O.beta_fgm(5)
    assert b[1] == 0.0
    # beta_2 = (theta_2 - 1)/theta_3 with theta_2 - 1 = (sqrt5 - 1)/2; S:236 prints 0.28172 (typo)
    assert b[2] == pytest.approx(((math.sqrt(5) - 1) / 2) / th[3], rel=1e-15)
    assert b[2] == pytest.approx(0.281753525125, abs=1e-11)


def test_fom_gm_single_step(golden):
    """GM on phi(u) = u^2 - 2u (L = 2), x0 = 0 -> x1 = 1 exactly."""
    ex = golden["fom_gm_step"]
    x = O.fom(lambda y: 2 * y - 2, np.array([ex["x0"]]), ex["L"], np.array([-10.0]),
              np.array([10.0]), 1, O.INNER_GM)
    assert x[0] == ex["x1"]


@pytest.mark.parametrize("rule,p", [(O.INNER_GM, 1), (O.INNER_FGM, 2)])
def test_fom_lemma1_envelope(rule, p):
    """Lemma 1: phi(x^k) - phi* <= 2 L R^2 / (k+1)^p on random box QPs,
    phi* and x* from brute-force enumeration (independent)."""
    for seed in range(4):
        prob = qpgen.tiny(5, 0, seed=seed, kind="ineq", box=0.6)
        Q, q = prob.Q, prob.q
        ref = kkt.brute_force(Q, q, np.zeros((0, 5)), np.zeros(0), prob.lb, prob.ub, np.zeros(0, np.uint8))
        L = float(np.linalg.eigvalsh(Q)[-1])
        x0 = np.full(5, 0.6) * np.sign(np.arange(5) - 2.0)
        R = np.linalg.norm(x0 - ref.u)
        hist = []
        O.fom(lambda y: Q @ y + q, x0, L, prob.lb, prob.ub, 200, rule, history=hist)
        for k, x in enumerate(hist, start=1):
            gap = 0.5 * x @ Q @ x + q @ x - ref.F
            assert gap <= 2 * L * R * R / (k + 1) ** p + 1e-12


# ------------------------------------------------------------------ DFOM steps
def test_dual_step_examples(golden):
    """one DFOM step lambda^1 = [mu^1 + grad/(2 L_d)]_{K_d}.
    Construction: G = 0, so grad_bar = g regardless of u (rho = 0, s = 0)."""
    for ex in golden["dual_step"]:
        g = _a(ex["grad"])
        res = O.dfom(np.eye(1), np.zeros(1), np.zeros((1, 1)), g, np.array([-1.0]), np.array([1.0]),
                     np.array(ex["cone"], np.uint8), 0.0, O.DGM, 1, 1, 1.0, ex["L_d"],
                     project_dual=ex["project_dual"])
        assert np.array_equal(res.lam, _a(ex["lam"])), ex["cite"]


def test_average_examples(golden):
    """S:349-350 (Eq. average_primal).  Construction: Q = 1, q = 0, G = 1 (ZERO row),
    rho = 0, L_in = 1, one GM inner step gives u_bar = -mu exactly; g = -4, L_d = 1 makes
    u_bar^1 = 0 and u_bar^2 = 2."""
    for ex in golden["average"]:
        res = O.dfom(np.eye(1), np.zeros(1), np.eye(1), np.array([-4.0]), np.array([-10.0]),
                     np.array([10.0]), np.array([0], np.uint8), 0.0, ex["alg"], 2, 1, 1.0, 1.0,
                     inner_rule=O.INNER_GM, keep_trace=True)
        assert np.array_equal(res.trace_u[0], [0.0]) and np.array_equal(res.trace_u[1], [2.0])
        if "out" in ex:
            assert res.x_avg[0] == pytest.approx(ex["out"][0], rel=1e-15), ex["cite"]
        else:
            assert res.x_avg[0] == pytest.approx(ex["out_approx"][0], abs=5e-4), ex["cite"]
            th2 = (1 + math.sqrt(5)) / 2
            assert res.x_avg[0] == pytest.approx(2 * th2 / (1 + th2), rel=1e-15)


def test_dfgm_weight_sum_is_theta_squared():
    """S_k = theta_k^2 for the DFGM averaging weights."""
    prob = qpgen.tiny(3, 2, seed=1)
    for K in (1, 2, 7, 40):
        res = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, O.DFGM,
                     K, 2, 10.0, 1.0)
        assert res.S == pytest.approx(O.theta_sequence(K)[K] ** 2, rel=1e-12)


def test_dgm_last_iterate_is_next_inner_solve():
    """for DGM the last iterate u_bar(lambda^k) coincides with u_bar^{k+1}
    (mu^{k+1} = lambda^k, same warm start) -- bit for bit."""
    prob = qpgen.tiny(6, 4, seed=4)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    a = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, O.DGM, 5, 4, L_in, L_d)
    b = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, O.DGM, 6, 4, L_in, L_d,
               keep_trace=True)
    assert np.array_equal(a.x_last, b.trace_u[5])


def test_lipschitz_ld_example(golden):
    """S:430 / Eq. (Ld): lambda_min = 1, rho = 0, ||G|| = 2 -> L_d = 4."""
    ex = golden["lipschitz_Ld"]
    G = np.array([[ex["normG"], 0.0]])
    Q = np.diag([ex["lambda_min"], 3.0])
    _, L_d, nG2 = O.lipschitz_constants(Q, G, ex["rho"], ex["lambda_min"])
    assert nG2 == pytest.approx(ex["normG"] ** 2) and L_d == pytest.approx(ex["L_d"])


# ---------------------------------------------------------------- brute force
def test_bruteforce_examples(golden):
    for ex in golden["bruteforce"]:
        n = len(ex["q"])
        G = _a(ex["G"]).reshape(-1, n)
        sol = kkt.brute_force(_a(ex["Q"]), _a(ex["q"]), G, _a(ex["g"]), _a(ex["lb"]), _a(ex["ub"]),
                              np.array(ex["cone"], np.uint8))
        assert np.allclose(sol.u, ex["u"], atol=1e-12), ex["cite"]
        assert sol.F == pytest.approx(ex["F"], abs=1e-12), ex["cite"]
        if "lam" in ex:
            assert np.allclose(sol.lam, ex["lam"], atol=1e-12), ex["cite"]


def test_kkt_equality_example_and_dfom_converges(golden):
    """u* = (1/2, 1/2), lambda* = -1/2 via the KKT linear solve; DFGM and DGM
    (rho = 1 and rho = 0) converge to it."""
    ex = golden["bruteforce"][1]
    Q, q, G, g = _a(ex["Q"]), _a(ex["q"]), _a(ex["G"]), _a(ex["g"])
    sol = kkt.kkt_equality(Q, q, G, g)
    assert np.allclose(sol.u, [0.5, 0.5]) and np.allclose(sol.lam, [-0.5])
    lb, ub, cone = _a(ex["lb"]), _a(ex["ub"]), np.array(ex["cone"], np.uint8)
    for rho, alg in ((1.0, O.DFGM), (0.0, O.DFGM), (1.0, O.DGM)):
        L_in, L_d, _ = O.lipschitz_constants(Q, G, rho, 1.0)
        res = O.dfom(Q, q, G, g, lb, ub, cone, rho, alg, 400, 50, L_in, L_d)
        assert np.allclose(res.x_last, sol.u, atol=1e-8)
        assert np.allclose(res.lam, sol.lam, atol=1e-7)


@pytest.mark.parametrize("kind", ["ineq", "mixed", "eq"])
@pytest.mark.parametrize("rho,alg", [(1.0, O.DFGM), (0.0, O.DFGM), (1.0, O.DGM), (4.0, O.DFGM)])
def test_dfom_reaches_bruteforce_optimum(kind, rho, alg):
    """Whole solve vs active-set enumeration: u* unique (Q > 0), so the
    last iterate must converge to it; lambda stays in K_d; F(x_avg) close too."""
    for seed in range(2):
        prob = qpgen.tiny(5, 3, seed=20 + seed, kind=kind, box=0.4)
        ref = kkt.brute_force(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone)
        lmin = float(np.linalg.eigvalsh(prob.Q)[0])
        L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, rho, lmin)
        outer = 400 if (alg == O.DFGM and rho > 0) else 4000
        res = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, alg,
                     outer, 40, L_in, L_d, keep_trace=True)
        tol = 2e-6 if rho > 0 else 1e-4      # rho = 0: slow dual (L_d = ||G||^2 / lambda_min(Q))
        assert np.allclose(res.x_last, ref.u, atol=tol), (seed, np.abs(res.x_last - ref.u).max())
        for lam in res.trace_lam:                       # lambda^k in K_d
            assert np.all(lam[prob.cone == qpgen.NONPOS] >= 0.0)
        F_avg = 0.5 * res.x_avg @ prob.Q @ res.x_avg + prob.q @ res.x_avg
        assert abs(F_avg - ref.F) <= 5e-2 * (1 + abs(ref.F))


def _box_qp_min(H, c, lb, ub):
    n = H.shape[0]
    return kkt.brute_force(H, c, np.zeros((0, n)), np.zeros(0), lb, ub, np.zeros(0, np.uint8))


def _exact_dual(prob, rho, mu):
    """d_rho(mu) exactly via enumeration: for rho = 0, or rho > 0 with K = {0}, L_rho(., mu)
    is a box QP."""
    Q, q, G, g = prob.Q, prob.q, prob.G, prob.g
    if rho == 0:
        sol = _box_qp_min(Q, q + G.T @ mu, prob.lb, prob.ub)
        return sol.F + mu @ g, sol.u
    assert np.all(prob.cone == qpgen.ZERO)
    H = Q + rho * G.T @ G
    c = q + G.T @ (mu + rho * g)
    sol = _box_qp_min(H, c, prob.lb, prob.ub)
    w = g + mu / rho
    const = 0.5 * rho * w @ w - mu @ mu / (2 * rho)
    return sol.F + const, sol.u


@pytest.mark.parametrize("alg,p_exp", [(O.DGM, 1), (O.DFGM, 2)])
@pytest.mark.parametrize("kind,rho", [("ineq", 0.0), ("eq", 1.0)])
def test_theorem1_and_weak_duality(alg, p_exp, kind, rho):
    """Theorem 1: F* - d(lambda^k) <= 4 L_d R_d^2/(k+1)^p + 2(k+1)^(p-1) eps_in,
    with d, eps_in = max_k L(u_bar^k, mu^k) - d(mu^k) (duquad_in) and F*, R_d = ||lambda*||
    from enumeration; weak duality d(lambda^k) <= F* (P:964)."""
    prob = qpgen.tiny(4, 2, seed=31, kind=kind, box=0.5)
    ref = kkt.brute_force(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone)
    lmin = float(np.linalg.eigvalsh(prob.Q)[0])
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, rho, lmin)
    K = 40
    res = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, alg, K, 30,
                 L_in, L_d, keep_trace=True)
    eps_in = 0.0
    for mu, u in zip(res.trace_mu, res.trace_u):
        d_mu, _ = _exact_dual(prob, rho, mu)
        Lval = O.aug_lagrangian(prob.Q, prob.q, prob.G, prob.g, prob.cone, rho, u, mu)
        assert Lval - d_mu >= -1e-10                      # left inequality of (duquad_in)
        eps_in = max(eps_in, Lval - d_mu)
    R_d = np.linalg.norm(ref.lam)
    for k, lam in enumerate(res.trace_lam, start=1):
        d_lam, _ = _exact_dual(prob, rho, lam)
        assert d_lam <= ref.F + 1e-10                     # weak duality
        bound = 4 * L_d * R_d ** 2 / (k + 1) ** p_exp + 2 * (k + 1) ** (p_exp - 1) * eps_in
        assert ref.F - d_lam <= bound + 1e-10, (k, ref.F - d_lam, bound)


def test_inexact_gradient_bound():
    """(inexact_gradient_rel) P:529-531: ||grad_bar d(mu) - grad d(mu)|| <= sqrt(2 L_d eps_in),
    with the exact u(mu) from enumeration (rho = 0, K = R_-: grad d = G u(mu) + g)."""
    prob = qpgen.tiny(5, 3, seed=8, kind="ineq", box=0.5)
    lmin = float(np.linalg.eigvalsh(prob.Q)[0])
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 0.0, lmin)
    rng = np.random.default_rng(0)
    for _ in range(10):
        mu = np.abs(rng.normal(size=prob.p))
        x0 = rng.uniform(-0.5, 0.5, prob.n)
        u_bar = O.inner_solve(prob.Q, prob.q, prob.G, prob.g, prob.cone, 0.0, mu, x0, L_in,
                              prob.lb, prob.ub, 3)
        d_mu, u_ex = _exact_dual(prob, 0.0, mu)
        eps_in = O.aug_lagrangian(prob.Q, prob.q, prob.G, prob.g, prob.cone, 0.0, u_bar, mu) - d_mu
        gbar = O.inexact_dual_grad(prob.G, prob.g, prob.cone, 0.0, u_bar, mu)
        gex = prob.G @ u_ex + prob.g
        assert np.linalg.norm(gbar - gex) <= math.sqrt(2 * L_d * max(eps_in, 0)) + 1e-9


# ------------------------------------------------------ batch / sparse forms
def test_batch_columns_match_single_runs():
    prob = qpgen.mpc_batch(6, seed=1, N=4)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    res = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, O.DFGM, 8, 5,
                 L_in, L_d)
    for b in range(6):
        r1 = O.dfom(prob.Q, prob.q[:, b], prob.G, prob.g[:, b], prob.lb, prob.ub, prob.cone, 1.0,
                    O.DFGM, 8, 5, L_in, L_d)
        assert np.allclose(res.x_last[:, b], r1.x_last, rtol=0, atol=1e-13)
        assert np.allclose(res.lam[:, b], r1.lam, rtol=0, atol=1e-12)


def test_sparse_matches_dense():
    import scipy.sparse as sp
    prob = qpgen.sparse_banded_eq(n=300, p=100, seed=3)
    Qd, Gd = prob.Q.toarray(), prob.G.toarray()
    # Gershgorin (docstring of sparse_banded_eq)
    ev = np.linalg.eigvalsh(Qd)
    assert ev[0] >= 0.5 - 1e-12 and ev[-1] <= 3.0 + 1e-12
    assert prob.Q.nnz == 300 + 2 * sum(300 - d for d in range(1, 6))
    L_in, L_d, _ = O.lipschitz_constants(Qd, Gd, 5.0, 0.5)
    a = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 5.0, O.DFGM, 5, 5, L_in, L_d)
    b = O.dfom(Qd, prob.q, Gd, prob.g, prob.lb, prob.ub, prob.cone, 5.0, O.DFGM, 5, 5, L_in, L_d)
    assert np.allclose(a.x_last, b.x_last, rtol=0, atol=1e-12)


def test_config0_matches_independent_solver():
    """Config 0 (BASELINE.json configs[0]): DFGM rho = 1, 200 x 50 reaches the optimum found by
    an independent NLP solver (SciPy SLSQP) -- |F - F*| and dist_K within 1e-6."""
    from scipy.optimize import minimize
    prob = qpgen.dense_ineq(50, 25, seed=0)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.1)
    res = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, O.DFGM, 200, 50,
                 L_in, L_d)
    cons = [dict(type="ineq", fun=lambda u: -(prob.G @ u + prob.g), jac=lambda u: -prob.G)]
    sl = minimize(lambda u: 0.5 * u @ prob.Q @ u + prob.q @ u, np.zeros(50),
                  jac=lambda u: prob.Q @ u + prob.q, bounds=[(-1, 1)] * 50, constraints=cons,
                  method="SLSQP", options=dict(ftol=1e-15, maxiter=1000))
    Fstar = sl.fun
    F = O.objective(prob.Q, prob.q, res.x_last)
    assert abs(F - Fstar) <= 1e-6 * (1 + abs(Fstar))
    assert O.dist_K(prob.G @ res.x_last + prob.g, prob.cone) <= 1e-6


def test_fgm_hand_worked_iterates():
    """FGM on phi(u) = u^2/2 with L = 2, x^0 = 1, worked by hand:
    x^1 = 1/2, y^2 = x^1 (beta_1 = 0), x^2 = 1/4,
    y^3 = x^2 + beta_2 (x^2 - x^1) = 0.25 - 0.25 * 0.2817535 = 0.1795616, x^3 = 0.0897808."""
    hist = []
    O.fom(lambda y: y, np.array([1.0]), 2.0, np.array([-5.0]), np.array([5.0]), 3, O.INNER_FGM,
          history=hist)
    assert hist[0][0] == 0.5 and hist[1][0] == 0.25
    assert hist[2][0] == pytest.approx(0.0897808, abs=1e-7)


def test_fgm_accelerates_over_gm():
    """Lemma 1: on an ill-conditioned box QP the FGM gap after 200 steps is far
    below the GM gap (rates 1/k^2 vs 1/k); a wrong momentum sign or index destroys this."""
    rng = np.random.default_rng(5)
    U, _ = np.linalg.qr(rng.normal(size=(8, 8)))
    Q = U @ np.diag(np.logspace(-4, 0, 8)) @ U.T
    q = rng.normal(size=8)
    lb, ub = -1e6 * np.ones(8), 1e6 * np.ones(8)
    ref = kkt.kkt_equality(Q, q, np.zeros((0, 8)), np.zeros(0))      # interior optimum
    assert np.all(np.abs(ref.u) < 1e6)
    gaps = {}
    for rule in (O.INNER_GM, O.INNER_FGM):
        x = O.fom(lambda y: Q @ y + q, np.zeros(8), 1.0, lb, ub, 200, rule)
        gaps[rule] = 0.5 * x @ Q @ x + q @ x - ref.F
    assert gaps[O.INNER_FGM] < 0.5 * gaps[O.INNER_GM]


# ---------------------------------------------------------------- NEXT-1: eps_in stopping, schedules
@pytest.mark.parametrize("kind,rho,eps_in", [("ineq", 0.0, 1e-4), ("ineq", 1.0, 1e-6), ("eq", 0.0, 1e-6),
                                             ("mixed", 2.0, 1e-5)])
def test_eps_inner_stop_meets_duquad_in(kind, rho, eps_in):
    """The gradient-map test of fom_run guarantees Eq. (duquad_in), P:445-451:
    L_rho(u_bar, mu) - d_rho(mu) <= eps_in, with d_rho(mu) from a 20000-step solve (which is
    within ~1e-13 of the minimum here, so the check is effectively against the exact value)."""
    prob = qpgen.tiny(8, 5, seed=11, kind=kind, shift=0.3)
    L_in, _, _ = O.lipschitz_constants(prob.Q, prob.G, rho, 0.1)
    sigma_L = float(np.linalg.eigvalsh(prob.Q)[0])     # <= lambda_min of the Hessian of L_rho(., mu)
    rng = np.random.default_rng(3)
    mu = rng.standard_normal(5) * 2.0
    x0 = O.clamp_U(np.zeros(8), prob.lb, prob.ub)
    info, gm = [], []
    ub = O.inner_solve(prob.Q, prob.q, prob.G, prob.g, prob.cone, rho, mu, x0, L_in, prob.lb, prob.ub, 5000,
                       eps_in=eps_in, sigma_L=sigma_L, gm=gm, info=info)
    k, conv = info[0]
    thr = np.sqrt(2 * sigma_L * eps_in)
    assert conv and k < 5000 and gm[-1] <= thr and all(v > thr for v in gm[:-1])
    d_rho, _ = O.dual_value(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, mu, L_in)
    gap = O.aug_lagrangian(prob.Q, prob.q, prob.G, prob.g, prob.cone, rho, ub, mu) - d_rho
    assert -1e-12 <= gap <= eps_in, gap
    # the fixed-count solve with the same number of steps is the same iterate
    same = O.inner_solve(prob.Q, prob.q, prob.G, prob.g, prob.cone, rho, mu, x0, L_in, prob.lb, prob.ub, k)
    assert np.array_equal(same, ub)


@pytest.mark.parametrize("alg", [O.DGM, O.DFGM])
@pytest.mark.parametrize("eps,R_d,L_d", [(1e-2, 1.0, 1.0), (1e-3, 3.7, 0.25), (0.5, 12.0, 40.0),
                                         (1e-4, 0.2, 7.5)])
def test_schedule_satisfies_theorem1_and_lemma1(alg, eps, R_d, L_d):
    """(choose_ein) is derived by making Theorem 1's bound (bound_gen_dfg)
    at most eps: evaluate that bound at (k_out, eps_in).  k_in comes from Lemma 1
    (bound_gen_dfg1) with R_phi <= D_U: evaluate Lemma 1 at k_in, both regimes."""
    for sigma_L, L_in, D_U in [(0.5, 40.0, 2.0), (0.0, 40.0, 2.0), (1e-3, 1e4, 1.0)]:
        s = O.theory_schedule(alg, eps, R_d, L_d, L_in, sigma_L, D_U, normG=3.0)
        assert O.theorem1_bound(alg, s["k_out"], L_d, R_d, s["eps_in"]) <= eps * (1 + 1e-12)
        assert O.lemma1_bound(s["k_in"], L_in, sigma_L, D_U, p=2) <= s["eps_in"] * (1 + 1e-12)
        # not wasteful: (choose_ein) takes k_out = q (DGM) / sqrt(q) (DFGM), q = 8 L_d R_d^2 / eps,
        # while the first term needs (k+1)^p >= q; two outer iterations fewer miss eps/2
        p = 1 if alg == O.DGM else 2
        assert s["k_out"] < 2 or 4 * L_d * R_d ** 2 / (s["k_out"] - 1) ** p >= eps / 2 * (1 - 1e-9)
        assert s["rho_star"] == pytest.approx(8 * R_d ** 2 / eps, rel=1e-15)
    assert O.theory_schedule(alg, eps, R_d, L_d, 40.0, 0.5, 2.0, 3.0, lambda_min_Q=0.1)["case_id"] == 1
    assert O.theory_schedule(alg, eps, R_d, L_d, 40.0, 0.5, 2.0, 3.0, lambda_min_Q=0.0)["case_id"] == 2
    # SPEC.md:412-414 classification examples, the eigenvalues from the matrices themselves:
    # Q = I -> Case 1; Q = 0 -> Case 2; Q = diag(1, 1e-12) -> Case 2 under tau_pd = 1e-7 lambda_max
    for Q, want in ((np.eye(3), 1), (np.zeros((3, 3)), 2), (np.diag([1.0, 1e-12]), 2), (np.diag([1e3, 2e-4]), 1),
                    (np.diag([1e3, 5e-5]), 2)):
        ev = np.linalg.eigvalsh(Q)
        got = O.theory_schedule(alg, eps, R_d, L_d, 40.0, 0.5, 2.0, 3.0, lambda_min_Q=max(ev[0], 0.0),
                                lambda_max_Q=ev[-1])["case_id"]
        assert got == want, (np.diag(Q), got)
    # ||G|| = 0 (no coupling): k_total = 0 rather than 0 * log(0)
    assert O.theory_schedule(alg, eps, R_d, L_d, 40.0, 0.5, 2.0, 0.0)["k_total"] == 0


@pytest.mark.parametrize("alg", [O.DGM, O.DFGM])
@pytest.mark.parametrize("seed", [21, 22])
def test_dfom_on_the_schedule_reaches_eps(alg, seed):
    """Theorem 1's conclusion: with eps_in and k_out from (choose_ein) and inner solves stopped at
    accuracy eps_in, F* - d_rho(lambda^{k_out}) <= eps (Case 1: Q > 0, rho = 0), with
    F* and R_d = ||lambda*|| from brute-force active-set enumeration (oracle.kkt)."""
    from oracle import kkt
    prob = qpgen.tiny(6, 4, seed=seed, kind="ineq", shift=1.0)
    G = 0.4 * prob.G
    g = 0.4 * prob.g
    ref = kkt.brute_force(prob.Q, prob.q, G, g, prob.lb, prob.ub, prob.cone)
    lmin = float(np.linalg.eigvalsh(prob.Q)[0])
    normG2 = float(np.linalg.eigvalsh(G.T @ G)[-1])
    L_in = float(np.linalg.eigvalsh(prob.Q)[-1])
    L_d = normG2 / lmin
    R_d = max(float(np.linalg.norm(ref.lam)), 1e-3)
    eps = 0.05
    s = O.theory_schedule(alg, eps, R_d, L_d, L_in, lmin, 2.0, np.sqrt(normG2), lmin)
    assert s["case_id"] == 1 and s["k_out"] <= 2000
    r = O.dfom(prob.Q, prob.q, G, g, prob.lb, prob.ub, prob.cone, 0.0, alg, s["k_out"], 100000, L_in, L_d,
               eps_in=s["eps_in"], sigma_L=lmin)
    assert all(r.converged)
    d, _ = O.dual_value(prob.Q, prob.q, G, g, prob.lb, prob.ub, prob.cone, 0.0, r.lam, L_in)
    assert ref.F - d <= eps, (ref.F - d, eps)
    assert ref.F - d >= -1e-9                       # weak duality


@pytest.mark.parametrize("alg", [O.DGM, O.DFGM])
def test_warm_start_at_the_kkt_point_is_a_fixed_point(alg):
    """Warm start (NEXT-2): started from u_bar^0 = u*, lambda^0 = lambda* (brute-force KKT,
    oracle.kkt) DFOM stays there -- the dual gradient G u(lambda*) + g - s vanishes at the
    optimum and u(lambda*) = u* -- while a cold start with the same budget has not
    converged; rho = 0 (Case 1, K_d = R^p_+)."""
    from oracle import kkt
    prob = qpgen.tiny(7, 4, seed=32, kind="ineq", shift=0.5)
    prob.q = 4.0 * prob.q                              # pushes the minimizer onto a constraint
    ref = kkt.brute_force(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone)
    assert np.max(ref.lam) > 1e-3                      # some constraint is active
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 0.0, float(np.linalg.eigvalsh(prob.Q)[0]))
    warm = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 0.0, alg, 3, 400, L_in, L_d,
                  x0=ref.u, lam0=ref.lam.copy())
    assert np.max(np.abs(warm.x_last - ref.u)) <= 1e-8
    assert np.max(np.abs(warm.lam - ref.lam)) <= 1e-8
    cold = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 0.0, alg, 3, 400, L_in, L_d)
    assert np.max(np.abs(cold.lam - ref.lam)) > 1e-4


# ------------------------------------------------------------ DGM dual averaging (NEXT-2)
def _eq_qp(n=12, p=5, seed=3):
    rng = np.random.default_rng(seed)
    R = rng.standard_normal((n, n))
    Q = 2.0 * np.eye(n) + 0.05 * (R + R.T)                 # kappa(Q) ~ 1.3: FGM converges to ulp fast
    G = rng.standard_normal((p, n))
    q, g = rng.standard_normal(n), rng.standard_normal(p)
    lb, ub = np.full(n, -np.inf), np.full(n, np.inf)       # no box: u_bar(mu) has a closed form
    cone = np.zeros(p, np.uint8)                           # equality rows: K = {0}, K_d = R^p
    return Q, q, G, g, lb, ub, cone


def test_dgm_dual_average_matches_the_closed_form_affine_recursion():
    """rho = 0, equality rows, no box: u_bar(mu) = -Q^{-1}(q + G'mu) and grad d(mu) = G u_bar(mu) + g,
    so DGM is the affine map lambda^{j} = lambda^{j-1} + (Gu_bar(lambda^{j-1}) + g) / (2 L_d).  The
    averaged final point of P:624-626 and its last iterate follow by plain linear algebra."""
    Q, q, G, g, lb, ub, cone = _eq_qp()
    Qi = np.linalg.inv(Q)
    H = G @ Qi @ G.T
    L_d = float(np.linalg.eigvalsh(H).max())
    L_in = float(np.linalg.eigvalsh(Q).max())
    ubar = lambda mu: -Qi @ (q + G.T @ mu)
    step = lambda lam: lam + (G @ ubar(lam) + g) / (2.0 * L_d)
    K = 7
    lams = [np.zeros(len(g))]
    for _ in range(K):
        lams.append(step(lams[-1]))
    lam_hat = np.mean(lams, axis=0)
    lam_fin = step(lam_hat)
    r = O.dfom(Q, q, G, g, lb, ub, cone, 0.0, O.DGM, K, 120, L_in, L_d, dual_average=True)
    assert np.allclose(r.lam_hat, lam_hat, rtol=0, atol=1e-11)
    assert np.allclose(r.lam, lam_fin, rtol=0, atol=1e-11)
    assert np.allclose(r.x_last, ubar(lam_fin), rtol=0, atol=1e-11)
    # and it is not the plain last dual iterate
    plain = O.dfom(Q, q, G, g, lb, ub, cone, 0.0, O.DGM, K, 120, L_in, L_d)
    assert np.allclose(plain.lam, lams[-1], rtol=0, atol=1e-11)
    assert np.max(np.abs(plain.lam - r.lam)) > 1e-6


def test_dgm_dual_average_final_point_in_Kd_and_dgm_only():
    prob = qpgen.tiny(30, 14, seed=2, kind="mixed", shift=0.3)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.2)
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, O.DGM, 6, 10, L_in, L_d,
               dual_average=True)
    nonpos = prob.cone == 1
    assert np.all(r.lam[nonpos] >= 0.0)
    assert r.lam_hat is not None and np.all(r.lam_hat[nonpos] >= 0.0)   # average of points of K_d
    assert len(r.inner_counts) == 0 or len(r.inner_counts) == 6 + 2
    with pytest.raises(ValueError):
        O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, O.DFGM, 6, 10, L_in, L_d,
               dual_average=True)


# ------------------------------------------------------------ bound diagnostics (NEXT-2)
@pytest.mark.parametrize("alg", ["DGM", "DFGM"])
def test_theory_bounds_hold_on_exact_inner_solves(alg):
    """Theorem 1, the drift bound and the last / average infeasibility
    bounds against actual DFOM runs on an equality QP with
    near-exact inner solves (eps_in ~ 0): lambda*, F* from the closed-form KKT system, d(lambda) in
    closed form (rho = 0, no box)."""
    Q, q, G, g, lb, ub, cone = _eq_qp(n=14, p=6, seed=5)
    sol = kkt.kkt_equality(Q, q, G, g)
    Qi = np.linalg.inv(Q)
    L_d = float(np.linalg.eigvalsh(G @ Qi @ G.T).max())
    L_in = float(np.linalg.eigvalsh(Q).max())
    R_d = float(np.linalg.norm(sol.lam))                 # lambda^0 = 0
    ubar = lambda mu: -Qi @ (q + G.T @ mu)
    dual = lambda lam: O.objective(Q, q, ubar(lam)) + lam @ (G @ ubar(lam) + g)
    for K in (1, 3, 10, 40):
        r = O.dfom(Q, q, G, g, lb, ub, cone, 0.0, alg, K, 120, L_in, L_d)
        gap = sol.F - dual(r.lam)
        assert -1e-9 <= gap <= O.theorem1_bound(alg, K, L_d, R_d, 0.0) + 1e-9
        assert np.linalg.norm(r.lam - sol.lam) <= O.drift_bound(K, L_d, R_d, 0.0) + 1e-9
        assert O.dist_K(G @ r.x_last + g, cone) <= O.feas_last_bound(alg, K, L_d, R_d, 0.0) + 1e-9
        assert O.dist_K(G @ r.x_avg + g, cone) <= O.feas_avg_bound(alg, K, L_d, R_d, 0.0) + 1e-9
    # the bounds are informative: at K = 40 they are below their K = 1 values
    assert O.feas_avg_bound(alg, 40, L_d, R_d, 0.0) < O.feas_avg_bound(alg, 1, L_d, R_d, 0.0)


def test_bound_formulas_special_values():
    """eps_in = 0 and R_d = 0 collapse every bound to 0 except the drift (R_d); DGM vs DFGM rates."""
    assert O.theorem1_bound("DGM", 9, 2.0, 0.0, 0.0) == 0.0
    assert O.feas_last_bound("DFGM", 9, 2.0, 0.0, 0.0) == 0.0
    assert O.drift_bound(9, 2.0, 3.0, 0.0) == 3.0
    assert O.drift_bound(9, 2.0, 0.0, 8.0) == pytest.approx(6.0)       # sqrt(9 * 8 / 2)
    assert O.feas_avg_bound("DGM", 4, 1.0, 1.0, 0.0) == pytest.approx(1.0)
    assert O.feas_avg_bound("DFGM", 4, 1.0, 1.0, 0.0) == pytest.approx(0.5)
    assert O.theorem1_bound("DFGM", 3, 1.0, 1.0, 0.0) == pytest.approx(4.0 / 16.0)
