# Config 1: session-start build (A) vs HEAD (B), alternated; then HEAD with the byte floor forced on
# at n = 2000 (DUQUAD_FUSED_NMIN=1000)
mkdir -p gpurun_out
c1() { timeout 600 python scripts/bench_configs.py --configs 1 2>/dev/null | python -c "
import json,sys
print(' '.join('%s/%g:%.2f' % (d['alg'], d['rho'], d['us_per_inner_step']) for d in map(json.loads, sys.stdin)))"; }
cp paper_1504_05708_b200/libduquad.so /tmp/keep.so
for i in 1 2; do for v in A B; do cp paper_1504_05708_b200/libduquad_$v.so paper_1504_05708_b200/libduquad.so; echo "$v $(c1)"; done; done | tee gpurun_out/c1_ab.txt
cp /tmp/keep.so paper_1504_05708_b200/libduquad.so
echo "B NMIN=1000 $(DUQUAD_FUSED_NMIN=1000 c1)" | tee -a gpurun_out/c1_ab.txt
