#!/usr/bin/env python
"""Config 4 (CSR, n = 1e6) pass timings for the sparse kernel variants (env overrides read at
setup: DUQUAD_SPK_A = 1 SELL / 2 thread-per-row for pass A, DUQUAD_LANE_UA / _UB = load-round
width, DUQUAD_PDL = 2 forces programmatic dependent launch, DUQUAD_DIA = 0 keeps banded Q rows in
SELL).  One JSON line per variant: us per inner step and per pass (CUDA events)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import qpgen
    from oracle import dfom as O  # noqa: F401  (not used: constants injected)
    from paper_1504_05708_b200 import Solver
    prob = qpgen.sparse_banded_eq()
    stream = torch.cuda.Stream()
    variants = [dict(), dict(DUQUAD_LANE_UA="8"), dict(DUQUAD_PDL="2"), dict(DUQUAD_DIA="0"), dict(),
                dict(sell=False)]
    for v in variants:
        for k in ("DUQUAD_SPK_A", "DUQUAD_LANE_UA", "DUQUAD_LANE_UB", "DUQUAD_PDL", "DUQUAD_DIA"):
            os.environ.pop(k, None)
        for k, x in v.items():
            if k.startswith("DUQUAD"):
                os.environ[k] = x
        s = Solver(prob.Q, prob.q, prob.G, prob.g, prob.lb, prob.ub, prob.cone, rho=5.0, lambda_min_lb=0.5,
                   stream=stream.cuda_stream, time_passes=True, sell_path=v.get("sell", True))
        s.set_constants(240.4, 0.1996)
        s.solve("DFGM", 20, 20)
        torch.cuda.synchronize()
        info = s.solve("DFGM", 60, 20)
        us = info["ms_device"] * 1e3 / info["inner_iters_total"]
        print(json.dumps(dict(variant=v, us_per_step=us, us_pass_a=info["ms_pass_a"] * 1e3,
                              us_pass_b=info["ms_pass_b"] * 1e3, kernels=info["sparse_kernels"])), flush=True)
        s.close()


if __name__ == "__main__":
    main()
