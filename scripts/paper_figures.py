"""The paper's experiments as GPU sweeps (qualitative reproduction only: the
figure values are not recoverable from the text and the comparison solvers are absent).

  fig2  P:657-673  primal suboptimality of DGM / DFGM vs the inner accuracy eps_in on a strongly
                   convex inequality QP, eps = 0.01, k_out from (choose_ein): DGM should be robust to
                   a coarse eps_in, DFGM sensitive.
  fig3  P:1372-1397 device time (ms) to reach |F(x_avg) - F*| <= eps and ||G x_avg + g|| <= eps on
                   random equality QPs (Q psd, K = {0}, rho = 1/eps) vs n: DGM with eps_in = eps,
                   DFGM with eps_in = 1e-3 and with the theory eps_in.
  fig4  P:1401-1423 outer iterations to reach |F - F*| <= eps and dist_K(Gu + g) <= eps in the last
                   and the average primal iterate on random inequality QPs (Q > 0), n = 10..500.

Everything runs through the public API (Solver, theory_schedule); F*, lambda* (R_d) come from long
DFGM reference solves on the GPU.  Iteration counts are searched on a geometric K grid, so they are
upper bounds at the grid's resolution.  Writes one JSON document (default profiles/r01_paper_figs.json).
  python scripts/paper_figures.py [--out FILE] [--quick]
"""
import argparse
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import qpgen
from paper_1504_05708_b200 import Solver, theory_schedule

EPS = 0.01
GRID = [1, 2, 3, 5, 8, 13, 21, 34, 55, 89, 144, 233, 377, 610, 987]


def reference(prob, rho, lmin):
    """F*, lambda*, constants from a long accurate DFGM solve."""
    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=rho, lambda_min_lb=lmin)
    L_in, L_d, nG2 = s.lipschitz(iters=150, safety=1e-6)
    s.solve("DFGM", 3000, 150)
    F, dist, _ = s.residuals("last")
    lam = s.result()[2]
    s.close()
    return dict(F=F, dist=dist, lam=lam, L_in=L_in, L_d=L_d, normG=float(np.sqrt(nG2)))


def meets(F, dist, Fs):
    return abs(F - Fs) <= EPS and dist <= EPS


def fig2(quick):
    n, p = (60, 30) if quick else (100, 50)
    prob = qpgen.dense_ineq(n, p, seed=7, shift=0.5)
    lmin = float(np.linalg.eigvalsh(prob.Q).min())
    ref = reference(prob, 0.0, lmin)
    R_d = max(float(np.linalg.norm(ref["lam"])), 1e-3)
    rows = []
    for alg in ("DGM", "DFGM"):
        sch = theory_schedule(alg, EPS, R_d, ref["L_d"], ref["L_in"], lmin, 2.0 * np.sqrt(n), ref["normG"], lmin)
        K = min(int(sch["k_out"]), 4000)
        for eps_in in (1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-6):
            s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=0.0, lambda_min_lb=lmin)
            s.set_constants(ref["L_in"], ref["L_d"])
            info = s.solve_eps(alg, K, 5000, eps_in, lmin)
            Fl, dl, _ = s.residuals("last")
            Fa, da, _ = s.residuals("avg")
            s.close()
            rows.append(dict(alg=alg, eps_in=eps_in, k_out=K, inner_total=int(info["inner_iters_total"]),
                             subopt_last=abs(Fl - ref["F"]), dist_last=dl, subopt_avg=abs(Fa - ref["F"]), dist_avg=da))
    return dict(n=n, p=p, eps=EPS, rows=rows)


def time_to_eps(prob, rho, lmin, ref, alg, eps_in, sigma_L):
    """(first K on the grid whose x_avg meets eps, device ms of that solve)"""
    for K in GRID:
        s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=rho, lambda_min_lb=lmin)
        s.set_constants(ref["L_in"], ref["L_d"])
        info = s.solve_eps(alg, K, 20000, eps_in, sigma_L)
        F, d, _ = s.residuals("avg")
        s.close()
        if meets(F, d, ref["F"]):
            return K, float(info["ms_device"])
    return None, None


def fig3(quick):
    rho = 1.0 / EPS
    out = []
    for n in ((20, 50) if quick else (20, 50, 100)):
        for inst in range(2 if quick else 3):
            prob = qpgen.tiny(n, n // 2, seed=1000 * n + inst, kind="eq", shift=0.0, psd_rank=max(1, n // 2))
            ref = reference(prob, rho, 1e-3)
            R_d = max(float(np.linalg.norm(ref["lam"])), 1e-3)
            th = theory_schedule("DFGM", EPS, R_d, ref["L_d"], ref["L_in"], 0.0, 2.0 * np.sqrt(n), ref["normG"], 0.0)
            for alg, e_in, tag in (("DGM", EPS, "DGM eps_in=eps"), ("DFGM", 1e-3, "DFGM eps_in=1e-3"),
                                   ("DFGM", th["eps_in"], "DFGM theory eps_in")):
                K, ms = time_to_eps(prob, rho, 1e-3, ref, alg, e_in, 1e-3)
                out.append(dict(n=n, instance=inst, variant=tag, eps_in=e_in, outer=K, ms=ms))
    return dict(eps=EPS, rho=rho, rows=out)


def fig4(quick):
    out = []
    for n in ((10, 50) if quick else (10, 50, 100, 200, 500)):
        for inst in range(3 if quick else 5):
            prob = qpgen.dense_ineq(n, max(1, n // 2), seed=5000 * n + inst, shift=0.5)
            lmin = float(np.linalg.eigvalsh(prob.Q).min())
            ref = reference(prob, 0.0, lmin)
            for alg in ("DGM", "DFGM"):
                first = {"last": None, "avg": None}
                for K in GRID:
                    s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=0.0,
                               lambda_min_lb=lmin)
                    s.set_constants(ref["L_in"], ref["L_d"])
                    s.solve(alg, K, 50)
                    for w in ("last", "avg"):
                        F, d, _ = s.residuals(w)
                        if first[w] is None and meets(F, d, ref["F"]):
                            first[w] = K
                    s.close()
                    if first["last"] is not None and first["avg"] is not None:
                        break
                out.append(dict(n=n, instance=inst, alg=alg, outer_last=first["last"], outer_avg=first["avg"]))
    return dict(eps=EPS, grid=GRID, rows=out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r01_paper_figs.json")
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    t0 = time.time()
    doc = dict(fig2=fig2(a.quick), fig3=fig3(a.quick), fig4=fig4(a.quick), wall_s=None)
    doc["wall_s"] = time.time() - t0
    with open(a.out, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps({k: (len(v["rows"]) if isinstance(v, dict) else v) for k, v in doc.items()}))


if __name__ == "__main__":
    main()
