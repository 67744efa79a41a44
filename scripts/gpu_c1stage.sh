# Dense pass kernels' y / w staging: plain loop (A, 38e63de) vs four loads in flight before the
# shared-memory stores (B, b79a71c): config 1 alternated A/B on one box
set -x
mkdir -p gpurun_out
c1() { timeout 600 python scripts/bench_configs.py --configs 1 2>/dev/null | python -c "
import json,sys
print(' '.join('%s/%g:%.2f' % (d['alg'], d['rho'], d['us_per_inner_step']) for d in map(json.loads, sys.stdin)))"; }
cp paper_1504_05708_b200/libduquad.so /tmp/keep.so
for i in 1 2 3; do for v in A B; do cp paper_1504_05708_b200/libduquad_$v.so paper_1504_05708_b200/libduquad.so; echo "$v $(c1)"; done; done | tee gpurun_out/c1_stage_ab.txt
cp /tmp/keep.so paper_1504_05708_b200/libduquad.so
