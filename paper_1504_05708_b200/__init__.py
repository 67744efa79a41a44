"""B200-native DuQuad hot path (arXiv 1504.05708): DGM / DFGM on sm_100a behind a C ABI.

The product path is `libduquad.so` (paper_1504_05708_b200/csrc, include/duquad.h);
this package is its thin ctypes binding.  No CPU fallback exists.
"""
from .solver import (Solver, nccl_unique_id, shard_range, solve_emulated, solve_emulated_eps,  # noqa: F401
                     theory_bounds, theory_schedule)
from ._lib import DuquadError  # noqa: F401
