"""Exact reference solutions for tiny QPs -- TEST INFRASTRUCTURE (see oracle/dfom.py header).

Used only to pin the oracle (tests/test_oracle_pins.py), never by the
product path.

* `kkt_equality`: closed-form KKT linear solve for equality-constrained QPs
  whose box is inactive: [Q G'; G 0][u; lam] = [-q; -g].
* `brute_force`: active-set enumeration (SPEC.md:479-487 design, n <= 10):
  every assignment {lower, upper, free} per coordinate and {active,
  inactive} per NONPOS row (ZERO rows always active); each assignment's
  equality-constrained KKT system is solved with numpy.linalg.lstsq, and the
  candidate is kept if it is primal feasible and its multipliers have the
  right signs.  Stationarity sign convention:
      Q u + q + G' lam - nu_lb + nu_ub = 0,  lam_i >= 0 on active NONPOS rows,
      nu >= 0 on active box faces,  matching the paper's Lagrangian
      F(u) + <lam, G u + g> with lam in K_d.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

ZERO = 0
NONPOS = 1


@dataclass
class KktSolution:
    u: np.ndarray
    lam: np.ndarray
    F: float
    kkt_residual: float


def kkt_equality(Q, q, G, g) -> KktSolution:
    n, p = Q.shape[0], G.shape[0]
    K = np.zeros((n + p, n + p))
    K[:n, :n] = Q
    K[:n, n:] = G.T
    K[n:, :n] = G
    rhs = np.concatenate([-q, -g])
    sol = np.linalg.solve(K, rhs)
    u, lam = sol[:n], sol[n:]
    F = 0.5 * u @ Q @ u + q @ u
    res = np.linalg.norm(Q @ u + q + G.T @ lam) + np.linalg.norm(G @ u + g)
    return KktSolution(u, lam, float(F), float(res))


def brute_force(Q, q, G, g, lb, ub, cone, tol=1e-9) -> KktSolution:
    n, p = Q.shape[0], G.shape[0]
    if n > 10:
        raise ValueError("brute force limited to n <= 10")
    nonpos_rows = [i for i in range(p) if cone[i] == NONPOS]
    zero_rows = [i for i in range(p) if cone[i] == ZERO]
    best = None
    for box_state in itertools.product((0, 1, 2), repeat=n):       # 0 free, 1 lower, 2 upper
        fixed = [j for j in range(n) if box_state[j] != 0]
        free = [j for j in range(n) if box_state[j] == 0]
        for act in itertools.product((0, 1), repeat=len(nonpos_rows)):
            rows = zero_rows + [nonpos_rows[t] for t in range(len(nonpos_rows)) if act[t]]
            u = np.zeros(n)
            for j in fixed:
                u[j] = lb[j] if box_state[j] == 1 else ub[j]
            nf, m = len(free), len(rows)
            # unknowns: u_free (nf), lam_rows (m)
            A = np.zeros((nf + m, nf + m))
            b = np.zeros(nf + m)
            Qff = Q[np.ix_(free, free)]
            A[:nf, :nf] = Qff
            if m:
                A[:nf, nf:] = G[np.ix_(rows, free)].T
                A[nf:, :nf] = G[np.ix_(rows, free)]
            b[:nf] = -(q[free] + Q[np.ix_(free, fixed)] @ u[fixed]) if nf else 0.0
            if m:
                b[nf:] = -(g[rows] + G[np.ix_(rows, fixed)] @ u[fixed])
            if nf + m:
                sol, *_ = np.linalg.lstsq(A, b, rcond=None)
                if np.linalg.norm(A @ sol - b) > 1e-8 * (1 + np.linalg.norm(b)):
                    continue
                u[free] = sol[:nf]
                lam_r = sol[nf:]
            else:
                lam_r = np.zeros(0)
            lam = np.zeros(p)
            lam[rows] = lam_r
            # primal feasibility
            if np.any(u < lb - tol) or np.any(u > ub + tol):
                continue
            r = G @ u + g
            if zero_rows and np.max(np.abs(r[zero_rows])) > 1e-7:
                continue
            if nonpos_rows and np.max(r[nonpos_rows]) > 1e-9:
                continue
            if any(lam[i] < -1e-9 for i in nonpos_rows):
                continue
            # box multipliers from stationarity
            s = Q @ u + q + G.T @ lam          # = nu_lb - nu_ub
            ok = True
            for j in range(n):
                if box_state[j] == 0 and abs(s[j]) > 1e-7 * (1 + np.abs(q).max()):
                    ok = False
                elif box_state[j] == 1 and s[j] < -1e-9:     # nu_lb = s >= 0
                    ok = False
                elif box_state[j] == 2 and s[j] > 1e-9:      # nu_ub = -s >= 0
                    ok = False
            if not ok:
                continue
            F = 0.5 * u @ Q @ u + q @ u
            if best is None or F < best.F - 1e-12:
                res = float(np.linalg.norm(np.where(np.array(box_state) == 0, s, 0.0)))
                best = KktSolution(u.copy(), lam.copy(), float(F), res)
    if best is None:
        raise RuntimeError("no feasible KKT point found")
    return best
