"""Stopping residuals every T outer iterations (duquad_solve_monitored, -m gpu).

The paper's stopping test: stop at the first checked outer
iteration j whose checked iterate u (x_last or x_avg) has |F(u) - F*| <= eps and dist_K(Gu + g)
<= eps; without a reference F*, the gap test |F(u) - d_bar(lambda^j)| <= eps (1 + |F(u)|) (reading
c24).  The per-check history (the SPEC trace fields) is checked value by value.  Checked against the oracle: the oracle's residuals at every checked j (dfom run for j
outer iterations) decide where the solve must stop; the GPU's returned iterates are bitwise a plain
solve(j); its reported F / dist match the oracle's at j to 1e-9."""
import math

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


def _oracle_checks(prob, rho, alg, T, jmax, Kin, L_in, L_d):
    """Per checked j = T, 2T, ..., jmax, straight from the oracle (dfom run for j outer
    iterations): F and dist_K of x_last and x_avg, and d_bar(lambda^j) = L_rho(x_last, lambda^j)."""
    out = []
    for j in range(T, jmax + 1, T):
        r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, alg, j, Kin, L_in, L_d)
        row = dict(k=j, dual_val=O.aug_lagrangian(prob.Q, prob.q, prob.G, prob.g, prob.cone, rho, r.x_last, r.lam))
        for tag, x in (("last", r.x_last), ("avg", r.x_avg)):
            row["f_" + tag] = O.objective(prob.Q, prob.q, x)
            row["infeas_" + tag] = float(O.dist_K(prob.G @ x + prob.g, prob.cone))
        out.append(row)
    return out


def _level(c, which, F_star):
    """The residual level the stopping test compares with eps (reading c24)."""
    F, d = c["f_" + which], c["infeas_" + which]
    obj = abs(F - F_star) if not math.isnan(F_star) else abs(F - c["dual_val"]) / (1 + abs(F))
    return max(obj, d)


def _eps_at(checks, j, which, F_star):
    """A tolerance the oracle's checked iterate meets at outer iteration j (1e-6 above its residual
    level, so no check sits within rounding of the threshold); never below 1e-10."""
    lvl = [_level(c, which, F_star) for c in checks]
    v = lvl[[c["k"] for c in checks].index(j)]
    if v < 1e-10:
        v = min(x for x in lvl if x >= 1e-10)
    return v * (1 + 1e-6)


def _first(checks, which, eps, F_star):
    return next(c["k"] for c in checks if _level(c, which, F_star) <= eps)


def _check_history(info, checks, Kin):
    for h in info["history"]:
        c = [c for c in checks if c["k"] == h["k"]][0]
        for key in ("dual_val", "f_last", "f_avg", "infeas_last", "infeas_avg"):
            assert abs(h[key] - c[key]) <= TOL * (1 + abs(c[key])), (key, h, c)
    ks = [h["k"] for h in info["history"]]
    assert ks == sorted(ks) and ks[-1] == info["outer_done"] and len(ks) == info["checks"]
    assert info["history"][-1]["inner_iters"] == info["inner_total"]


def _run(prob, rho, alg, Kmax, Kin, T, which, eps, F_star, L_in, L_d, **kw):
    from paper_1504_05708_b200 import Solver
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=rho, **kw)
    s.set_constants(L_in, L_d)
    info = s.solve_monitored(alg, Kmax, Kin, T, which, eps, F_star)
    got = s.result()
    st = s.get_state()
    s.close()
    t = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=rho, **kw)
    t.set_constants(L_in, L_d)
    t.solve(alg, info["outer_done"], Kin)
    plain = t.result()
    t.close()
    return info, got, plain, st


@pytest.mark.parametrize("which", ["last", "avg"])
@pytest.mark.parametrize("alg", ["DGM", "DFGM"])
def test_monitored_stops_at_the_oracles_first_pass(torch_cuda, alg, which):
    prob = qpgen.dense_ineq(50, 25, seed=0)
    rho, Kin, T, Kmax = 1.0, 10, 4, 120
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, rho, 0.1)
    ref = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho, "DFGM", 600, 50, L_in, L_d)
    F_star = O.objective(prob.Q, prob.q, ref.x_last)
    checks = _oracle_checks(prob, rho, alg, T, Kmax, Kin, L_in, L_d)
    eps = _eps_at(checks, 40, which, F_star)   # the oracle's residual level at j = 40: stops mid-run
    first = _first(checks, which, eps, F_star)
    info, got, plain, st = _run(prob, rho, alg, Kmax, Kin, T, which, eps, F_star, L_in, L_d, small_path=False)
    assert info["converged"] and info["outer_done"] == first and info["checks"] == first // T
    for a, b in zip(got, plain):
        assert np.array_equal(a, b)
    _check_history(info, checks, Kin)
    assert info["inner_total"] == (first + first // T) * Kin    # each segment adds its last-iterate solve
    assert st["outer_done"] == first


def test_monitored_cap_and_gap_test(torch_cuda, tmp_path):
    """Unreachable eps: every check fails, the solve runs to outer_max (a ragged last segment);
    F_star = NaN: the primal-dual gap test |F - d_bar(lambda^j)| <= eps (1 + |F|) with dist_K;
    the history exports as the SPEC trace CSV."""
    prob = qpgen.tiny(37, 13, seed=5, kind="mixed", shift=0.2)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 2.0, 0.2)
    info, got, plain, _ = _run(prob, 2.0, "DFGM", 11, 6, 4, "last", 1e-15, 0.0, L_in, L_d, small_path=False)
    assert not info["converged"] and info["outer_done"] == 11 and info["checks"] == 3
    for a, b in zip(got, plain):
        assert np.array_equal(a, b)
    checks = _oracle_checks(prob, 2.0, "DFGM", 5, 30, 6, L_in, L_d)
    for which in ("last", "avg"):
        eps = _eps_at(checks, 15, which, float("nan"))
        first = _first(checks, which, eps, float("nan"))
        info, got, plain, _ = _run(prob, 2.0, "DFGM", 30, 6, 5, which, eps, float("nan"), L_in, L_d,
                                   small_path=False)
        assert info["converged"] and info["outer_done"] == first
        for a, b in zip(got, plain):
            assert np.array_equal(a, b)
        _check_history(info, checks, 6)
    from paper_1504_05708_b200 import Solver
    Solver.write_trace_csv(tmp_path / "trace.csv", info["history"])
    lines = (tmp_path / "trace.csv").read_text().splitlines()
    assert lines[0] == "k,dual_val,f_last,f_avg,infeas_last,infeas_avg,inner_iters,cum_matvecs"
    assert len(lines) == 1 + info["checks"] and float(lines[1].split(",")[2]) == info["history"][0]["f_last"]


@pytest.mark.parametrize("kw", [dict(), dict(nccl_self=True)])
def test_monitored_byte_floor(torch_cuda, kw):
    """n >= 4096: the byte-floor path (single GPU, and the row-sharded schedule on real NCCL)."""
    prob = qpgen.dense_ineq(4096, 2048, seed=1, shift=0.05)
    L_in, L_d, _ = O.lipschitz_constants(prob.Q, prob.G, 1.0, 0.05)
    checks = _oracle_checks(prob, 1.0, "DFGM", 2, 8, 3, L_in, L_d)
    eps = _eps_at(checks, 6, "last", float("nan"))
    first = _first(checks, "last", eps, float("nan"))
    info, got, plain, _ = _run(prob, 1.0, "DFGM", 8, 3, 2, "last", eps, float("nan"), L_in, L_d, **kw)
    assert info["path"] in (1, 3) and info["converged"] and info["outer_done"] == first
    r = O.dfom(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, 1.0, "DFGM", first, 3, L_in, L_d)
    for a, b in zip(got, (r.x_last, r.x_avg, r.lam)):
        assert relerr(a, b) <= TOL
    if not kw:   # single GPU: bitwise a plain solve(first)
        for a, b in zip(got, plain):
            assert np.array_equal(a, b)


def test_monitored_rejects_bad_arguments(torch_cuda):
    from paper_1504_05708_b200 import Solver, DuquadError
    prob = qpgen.dense_ineq(50, 25, seed=0)
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0)
    s.set_constants(100.0, 1.0)
    for args in [(0, 5, 1, "avg", 1e-3), (10, 5, 0, "avg", 1e-3), (10, 5, 2, "avg", 0.0), (10, 5, 2, "avg", -1.0)]:
        with pytest.raises(DuquadError):
            s.solve_monitored("DFGM", args[0], args[1], args[2], args[3], args[4])
    with pytest.raises(DuquadError):
        s.solve_monitored("DFGM", 10, 5, 2, "avg", 1e-3, float("inf"))
    s.close()
    d = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=1.0, dual_average=True)
    d.set_constants(100.0, 1.0)
    with pytest.raises(DuquadError):
        d.solve_monitored("DGM", 10, 5, 2, "avg", 1e-3)
    d.close()


@pytest.mark.parametrize("case", ["csr", "rho0", "eq_h"])
def test_monitored_other_paths(torch_cuda, case):
    """The CSR, rho = 0 (K3) and equality-H paths: stop where the oracle's checks say, iterates bitwise
    a plain solve(j), history rows equal to the oracle's."""
    if case == "csr":
        prob, rho, lmin, kw = qpgen.sparse_banded_eq(n=3001, p=1201, seed=4), 5.0, 0.5, {}
        Qd, Gd = prob.Q.toarray(), prob.G.toarray()
    elif case == "rho0":
        prob, rho, lmin, kw = qpgen.dense_ineq(600, 300, seed=2, shift=0.1), 0.0, 0.1, dict(small_path=False)
        Qd, Gd = prob.Q, prob.G
    else:
        prob, rho, lmin, kw = qpgen.tiny(500, 150, seed=14, kind="eq"), 1.0, 0.2, dict(small_path=False)
        Qd, Gd = prob.Q, prob.G
    L_in, L_d, _ = O.lipschitz_constants(Qd, Gd, rho, lmin)
    T, Kmax, Kin = 2, 12, 5
    checks = _oracle_checks(prob, rho, "DFGM", T, Kmax, Kin, L_in, L_d)
    eps = _eps_at(checks, 8, "avg", float("nan"))
    first = _first(checks, "avg", eps, float("nan"))
    info, got, plain, _ = _run(prob, rho, "DFGM", Kmax, Kin, T, "avg", eps, float("nan"), L_in, L_d, **kw)
    assert info["path"] == {"csr": 5, "rho0": 2, "eq_h": 8}[case], info["path"]
    assert info["converged"] and info["outer_done"] == first
    for a, b in zip(got, plain):
        assert np.array_equal(a, b)
    _check_history(info, checks, Kin)
