"""Stress the two tests that failed once each (warm start, CSR / sharded byte floor) in ONE process,
interleaved with memory-heavy tests (device-memory reuse), and report every failure."""
import sys
import traceback
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import torch
import test_gpu_warm as W
import test_gpu_sharded as S
import test_gpu_csr as CSR
import qpgen

fails = {}
def run(name, fn, *a):
    try:
        fn(*a)
        return True
    except Exception as e:
        fails[name] = fails.get(name, 0) + 1
        print("FAIL", name, repr(e)[:300], flush=True)
        return False

c4 = qpgen.sparse_banded_eq()
for it in range(12):
    run("warm_csr", W.test_warm_start_csr, torch)
    run("sharded_floor_warm", S.test_sharded_byte_floor_ragged_warm_start_and_dual_average, torch)
    if it % 3 == 0:
        run("c2_8way", S.test_config2_full_size_8_way_sharding, torch)
        run("c4_full", CSR.test_config4_full_size_prefix, torch, c4)
    run("warm_dense_all", lambda t: [f(t) for n, f in vars(W).items() if n.startswith("test_") and "csr" not in n and "batched" not in n and f.__code__.co_argcount == 1], torch)
print("failures:", fails, flush=True)
