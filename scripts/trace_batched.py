"""Per-block timeline of CTA 0 of the batched pass-A kernel (instrumentation build):
    DUQUAD_NVCC_EXTRA=-DDUQUAD_BATCHED_TRACE python -c "from paper_1504_05708_b200 import build; build.build()"
    python scripts/trace_batched.py     # prints, per pass-A launch and 128-row block, globaltimer
columns (us from block 0), pass A: block start, K loop done, epilogue done, h tile ready, h-stager start /
done, ring producer first chunk, in-place pass done; pass B: group start, K loop done, C tile slot free,
-, epilogue start, epilogue done, producer first chunk.  Rebuild without the define afterwards."""
import sys; sys.path.insert(0, ".")
import qpgen
from paper_1504_05708_b200 import Solver
from oracle import dfom as O
prob = qpgen.mpc_batch(8192, seed=0)
s = Solver(prob.Q, prob.q.T.copy(), prob.G, prob.g.T.copy(), prob.lb, prob.ub, prob.cone, rho=1.0, use_graphs=False)
s.set_constants(600000.0, 1.0)
s.solve("DFGM", 1, 3)
