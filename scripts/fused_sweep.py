#!/usr/bin/env python
"""Tuning sweep of the byte-floor stream kernel at config 2: device time of one launch (CUDA
events on the library stream, time_passes) vs the Q/G role split (argv[1]: list of
DUQUAD_FUSED_NQ values, 0 = the library's default), the Q-only (rho = 0) kernel for each row-step
cost of the partition (env ROWCOSTS -> DUQUAD_FUSED_ROWCOST) and the two-pass reference.
Prints one JSON line per case."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import qpgen
    from paper_1504_05708_b200 import Solver
    nqs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,2,40,60,74,90,110,148").split(",")]
    n, p = 16384, 8192
    d = qpgen.dense_ineq_torch(n, p, seed=0, shift=0.05)
    st = torch.cuda.Stream()
    tri, gb = 8.0 * n * (n + 1) / 2, 8.0 * n * p

    def run(rho, fused, nq):
        if nq:
            os.environ["DUQUAD_FUSED_NQ"] = str(nq)
        else:
            os.environ.pop("DUQUAD_FUSED_NQ", None)
        s = Solver(d["Q"], d["q"], d["G"], d["g"], d["lb"], d["ub"], d["cone"], rho=rho, lambda_min_lb=0.05,
                   stream=st.cuda_stream, time_passes=True, fused_path=fused)
        s.set_constants(47588.0, 1.0)
        s.solve("DFGM", 2, 5)
        info = s.solve("DFGM", 3, 10)
        s.close()
        return info

    for nq in nqs:
        i = run(1.0, True, nq)
        print(json.dumps({"case": "fused", "nq": nq, "ms_stream": i["ms_pass_a"], "ms_epi": i["ms_pass_b"],
                          "floor_gbs": (tri + gb) / i["ms_pass_a"] / 1e6,
                          "it_s": i["inner_iters_total"] / (i["ms_device"] / 1e3)}), flush=True)
    for rc in os.environ.get("ROWCOSTS", "6144").split(","):
        os.environ["DUQUAD_FUSED_ROWCOST"] = rc
        i = run(0.0, True, 0)
        print(json.dumps({"case": "fused_rho0_q_only", "rowcost": float(rc), "ms_stream": i["ms_pass_a"],
                          "ms_epi": i["ms_pass_b"], "q_gbs": tri / i["ms_pass_a"] / 1e6}), flush=True)
    os.environ.pop("DUQUAD_FUSED_ROWCOST", None)
    i = run(1.0, False, 0)
    print(json.dumps({"case": "two_pass", "ms_a": i["ms_pass_a"], "ms_b": i["ms_pass_b"],
                      "it_s": i["inner_iters_total"] / (i["ms_device"] / 1e3)}), flush=True)


if __name__ == "__main__":
    main()
