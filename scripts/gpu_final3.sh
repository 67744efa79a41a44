# Final round-2 checkpoint after the config-4 slice interleave and the setup changes: full GPU tests,
# smoke, default bench, per-config bench, config-4 SELL load-round width 8 vs 4 under the interleave
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python scripts/bench_brief.py < gpurun_out/bench.json
timeout 900 python scripts/bench_configs.py --configs 0,1,3,4 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
for i in 1 2; do for u in 4 8; do
  echo "UA=$u $(DUQUAD_LANE_UA=$u timeout 300 python scripts/bench_configs.py --configs 4 --cases 1 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["us_per_inner_step"],2), round(1e3*d["ms_pass_a"],1), round(1e3*d["ms_pass_b"],1))')"
done; done | tee gpurun_out/c4_ua.txt
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"
