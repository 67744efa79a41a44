#!/usr/bin/env python
"""Per-config measurements of every §8(a) path on one B200 (companion of bench.py, which times
config 2 only).  Prints one JSON object per config: inner iterations/s, solves/s, device ms per
solve, and the achieved bandwidth / flop rate of the pass kernels from CUDA events.

  python scripts/bench_configs.py [--configs 0,1,3,4] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="0,1,3,4")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cases", type=int, default=99, help="max cases per config")
    args = ap.parse_args()
    import numpy as np
    import torch

    import qpgen
    from paper_1504_05708_b200 import Solver

    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    runs = []
    for c in [int(x) for x in args.configs.split(",")]:
        if c in (0, 1):
            n, p = (50, 25) if c == 0 else (2000, 1000)
            prob = qpgen.dense_ineq(n, p, seed=0)
            mk = lambda rho: Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=rho,
                                    lambda_min_lb=0.1, stream=stream.cuda_stream, time_passes=True)
            cases = [("DFGM", 1.0, 200, 50)] if c == 0 else [("DFGM", 1.0, 400, 50), ("DGM", 1.0, 400, 50),
                                                              ("DFGM", 0.0, 400, 20), ("DFGM", 10.0, 300, 200)]
        elif c == 3:
            prob = qpgen.mpc_batch(8192, seed=0)
            mk = lambda rho: Solver(prob.Q, prob.q.T.copy(), prob.G, prob.g.T.copy(), prob.lb, prob.ub, prob.cone,
                                    rho=rho, lambda_min_lb=0.1, stream=stream.cuda_stream, time_passes=True)
            cases = [("DFGM", 1.0, 50, 20)]
        elif c == 4:
            prob = qpgen.sparse_banded_eq()
            mk = lambda rho: Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=rho,
                                    lambda_min_lb=0.5, stream=stream.cuda_stream, time_passes=True)
            cases = [("DFGM", 5.0, 300, 50), ("DGM", 5.0, 300, 20)]
        for alg, rho, K, Kin in cases[:args.cases]:
            s = mk(rho)
            L_in, L_d, nG2 = s.lipschitz(iters=80, safety=1e-3)
            s.solve(alg, K, Kin)                       # warm-up (graph build, clocks)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.nvtx.range_push("timed")
            e0.record(stream)
            infos = [s.solve(alg, K, Kin) for _ in range(args.reps)]
            e1.record(stream)
            torch.cuda.nvtx.range_pop()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.reps
            i = infos[-1]
            inner = (K + 1) * Kin
            out = dict(config=c, alg=alg, rho=rho, outer=K, inner=Kin, ms_per_solve=ms,
                       inner_iters_per_s=inner / (ms / 1e3), solves_per_s=1e3 / ms,
                       us_per_inner_step=ms * 1e3 / inner, ms_pass_a=i["ms_pass_a"], ms_pass_b=i["ms_pass_b"],
                       L_in=L_in, L_d=L_d)
            if i["flops_pass_a"] > 0 and i["ms_pass_a"] > 0:
                out["tflops_pass_a"] = i["flops_pass_a"] / (i["ms_pass_a"] / 1e3) / 1e12
                out["tflops_pass_b"] = i["flops_pass_b"] / (i["ms_pass_b"] / 1e3) / 1e12
                out["tflops_step"] = (i["flops_pass_a"] + i["flops_pass_b"]) / (ms / 1e3 / inner) / 1e12
                out["qp_solves_per_s"] = 8192 * 1e3 / ms
            if i["ms_pass_a"] > 0:
                out["gbs_pass_a"] = i["bytes_pass_a"] / (i["ms_pass_a"] / 1e3) / 1e9
                out["gbs_pass_b"] = i["bytes_pass_b"] / (i["ms_pass_b"] / 1e3) / 1e9
                out["frac_pass_a_of_hbm"] = out["gbs_pass_a"] / peak
            out["kernel_launches"] = i["kernel_launches"]
            xl, xa, lam = s.result()
            if c != 3:
                F, dist, lag = s.residuals("last")
                out.update(F_last=F, dist_last=dist, lag_last=lag)
                Fa, da, _ = s.residuals("avg")
                out.update(F_avg=Fa, dist_avg=da)
            s.close()
            print(json.dumps(out), flush=True)
            runs.append(out)


if __name__ == "__main__":
    main()
