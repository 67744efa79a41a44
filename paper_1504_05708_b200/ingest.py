"""Two-sided linear constraints  lb_bar <= G_bar u + g_bar <= ub_bar ingested
into the form the solver takes, G u + g in K with a per-row cone tag (ZERO: = 0, NONPOS: <= 0).
Host-side argument preparation (S:122-130 gives the same rule):

  lb_bar_i == ub_bar_i            -> one ZERO row     G_bar_i u + (g_bar_i - ub_bar_i)  = 0
  lb_bar_i <  ub_bar_i            -> up to two NONPOS rows, infinite sides omitted:
                                      G_bar_i u + (g_bar_i - ub_bar_i) <= 0   (if ub_bar_i < inf)
                                     -G_bar_i u + (lb_bar_i - g_bar_i) <= 0   (if lb_bar_i > -inf)
  lb_bar_i > ub_bar_i or NaN      -> ValueError (infeasible / malformed specification)

`raw_multipliers` maps the solver's multipliers back to one per raw row: the multiplier of the
interval constraint is lambda_upper - lambda_lower (the ZERO row's multiplier as it is).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ZERO, NONPOS = 0, 1


@dataclass
class Ingested:
    G: object            # (p x n) ndarray, or scipy.sparse CSR if G_bar was sparse
    g: np.ndarray        # (p,)
    cone: np.ndarray     # (p,) uint8
    row: np.ndarray      # (p,) raw row index of each ingested row
    sign: np.ndarray     # (p,) +1 (ZERO or upper side), -1 (lower side)


def two_sided(G_bar, g_bar, lb_bar, ub_bar) -> Ingested:
    g_bar = np.asarray(g_bar, np.float64)
    lb_bar = np.asarray(lb_bar, np.float64)
    ub_bar = np.asarray(ub_bar, np.float64)
    m = g_bar.shape[0]
    if G_bar.shape[0] != m or lb_bar.shape != (m,) or ub_bar.shape != (m,):
        raise ValueError("G_bar, g_bar, lb_bar, ub_bar: inconsistent row counts")
    if np.isnan(g_bar).any() or np.isnan(lb_bar).any() or np.isnan(ub_bar).any():
        raise ValueError("NaN in the constraint data")
    dense = not hasattr(G_bar, "tocsr")
    if dense and np.isnan(np.asarray(G_bar, np.float64)).any():
        raise ValueError("NaN in G_bar")
    if (lb_bar > ub_bar).any():
        raise ValueError(f"lb_bar > ub_bar on rows {np.flatnonzero(lb_bar > ub_bar)[:8].tolist()}: "
                         "infeasible specification")
    rows, signs, gs, cones = [], [], [], []
    for i in range(m):
        lo, hi = lb_bar[i], ub_bar[i]
        if lo == hi:
            rows.append(i), signs.append(1.0), gs.append(g_bar[i] - hi), cones.append(ZERO)
            continue
        if np.isfinite(hi):
            rows.append(i), signs.append(1.0), gs.append(g_bar[i] - hi), cones.append(NONPOS)
        if np.isfinite(lo):
            rows.append(i), signs.append(-1.0), gs.append(lo - g_bar[i]), cones.append(NONPOS)
    row = np.asarray(rows, np.int64)
    sign = np.asarray(signs)
    if dense:
        G = np.asarray(G_bar, np.float64)[row] * sign[:, None]
    else:
        import scipy.sparse as sp
        G = (sp.diags(sign) @ G_bar.tocsr()[row]).tocsr()
        G.sort_indices()
    return Ingested(G, np.asarray(gs, np.float64), np.asarray(cones, np.uint8), row, sign)


def raw_multipliers(lam, ing: Ingested, m: int) -> np.ndarray:
    """One multiplier per raw row: sum of sign * lambda over the row's ingested rows (last axis)."""
    lam = np.asarray(lam, np.float64)
    out = np.zeros(lam.shape[:-1] + (m,))
    for k in range(lam.shape[-1]):
        out[..., ing.row[k]] += ing.sign[k] * lam[..., k]
    return out
