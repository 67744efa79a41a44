# Dense pass kernels with the matrix prefetch before griddepcontrol.wait (B) vs without (A):
# parity tests of the dense paths, then config 1 alternated A/B
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_state.py tests/test_gpu_warm.py -m gpu -x -q > gpurun_out/pytest_pre.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_pre.log
c1() { timeout 600 python scripts/bench_configs.py --configs 1 2>/dev/null | python -c "
import json,sys
print(' '.join('%s/%g:%.2f' % (d['alg'], d['rho'], d['us_per_inner_step']) for d in map(json.loads, sys.stdin)))"; }
cp paper_1504_05708_b200/libduquad.so /tmp/keep.so
for i in 1 2 3; do for v in A B; do cp paper_1504_05708_b200/libduquad_$v.so paper_1504_05708_b200/libduquad.so; echo "$v $(c1)"; done; done | tee gpurun_out/c1_pre_ab.txt
cp /tmp/keep.so paper_1504_05708_b200/libduquad.so
