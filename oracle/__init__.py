"""CPU oracle for the DuQuad DGM/DFGM hot path -- TEST INFRASTRUCTURE ONLY.

May be imported only by `tests/`, `__graft_entry__.smoke()` and `bench.py`
(cpu_baseline and --impl reference legs).  Shares no code with the CUDA
path.  Submodules: `oracle.dfom` (the algorithm, with citations) and
`oracle.kkt` (exact tiny-QP solutions used to pin it).
"""
