# K4 small kernel: short-column loads up front (B) vs looped (A); small-path GPU tests, then config 0
# alternated A/B (time per inner step and the final objective values, which must agree bitwise)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "small or warm or state or eps or dual_average or monitored" > gpurun_out/pytest_small.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_small.log
c0() { timeout 300 python scripts/bench_configs.py --configs 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['us_per_inner_step'],3), repr(d['F_last']), repr(d['F_avg']), repr(d['dist_avg']))"; }
cp paper_1504_05708_b200/libduquad.so /tmp/keep.so
for i in 1 2 3; do for v in A B; do cp paper_1504_05708_b200/libduquad_$v.so paper_1504_05708_b200/libduquad.so; echo "$v $(c0)"; done; done | tee gpurun_out/c0_short_ab.txt
cp /tmp/keep.so paper_1504_05708_b200/libduquad.so
