"""Timing of the byte-floor stream kernel per role split (tuning experiment; results invalid
for nq overrides that leave rows unprocessed)."""
import os, sys, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
code = r'''
import sys, json, torch
sys.path.insert(0, "%s")
import qpgen
from paper_1504_05708_b200 import Solver
d = qpgen.dense_ineq_torch(16384, 8192, seed=0, shift=0.05)
st = torch.cuda.Stream()
s = Solver(d["Q"], d["q"], d["G"], d["g"], d["lb"], d["ub"], d["cone"], rho=1.0, stream=st.cuda_stream, time_passes=True, use_graphs=False)
s.set_constants(47588.0, 1.0)
s.solve("DFGM", 2, 10)
i = s.solve("DFGM", 3, 20)
print(json.dumps(dict(nq=%s, ms_a=i["ms_pass_a"], ms_b=i["ms_pass_b"], bytes_a=i["bytes_pass_a"])))
''' 
for nq in ["74", "148", "0", "60", "88"]:
    env = dict(os.environ, DUQUAD_FUSED_NQ=nq)
    out = subprocess.run([sys.executable, "-c", code % (ROOT, nq)], env=env, capture_output=True, text=True)
    print(out.stdout.strip() or out.stderr[-500:], flush=True)
