"""Host-side phase times of one end-to-end config-2 solve through the public API from pinned host
buffers (the bench's e2e leg): setup (validation, upload, pack / transpose, symmetry check, path
choice), Lipschitz constants, solve, result copy, close."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import qpgen  # noqa: E402
from paper_1504_05708_b200 import Solver  # noqa: E402

torch.cuda.set_device(0)
d = qpgen.dense_ineq_torch(16384, 8192, seed=0, shift=0.05, device="cuda:0")
hp = {k: v.cpu().pin_memory() for k, v in d.items()}
del d
torch.cuda.empty_cache()
outer = int(os.environ.get("E2E_OUTER", "100"))
for rep in range(3):
    t = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = Solver(hp["Q"], hp["q"], hp["G"], hp["g"], hp["lb"], hp["ub"], hp["cone"], rho=1.0, lambda_min_lb=0.05)
    torch.cuda.synchronize(); t["setup"] = time.perf_counter() - t0; t0 = time.perf_counter()
    s.lipschitz(iters=60, safety=1e-3)
    torch.cuda.synchronize(); t["lipschitz"] = time.perf_counter() - t0; t0 = time.perf_counter()
    s.solve("DFGM", outer, 100)
    torch.cuda.synchronize(); t["solve"] = time.perf_counter() - t0; t0 = time.perf_counter()
    s.result()
    torch.cuda.synchronize(); t["result"] = time.perf_counter() - t0; t0 = time.perf_counter()
    s.close()
    torch.cuda.synchronize(); t["close"] = time.perf_counter() - t0
    print(json.dumps({k: round(v, 4) for k, v in t.items()}))
