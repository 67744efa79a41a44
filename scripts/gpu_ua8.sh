# SELL pass A load-round width with DIA Q rows: default (8) vs DUQUAD_LANE_UA=4, alternated; CSR tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_csr.py tests/test_gpu_sharded.py -m gpu -x -q > gpurun_out/pytest_ua8.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ua8.log
for i in 1 2 3; do for u in 4 default; do
  E=""; [ $u = 4 ] && E="DUQUAD_LANE_UA=4"
  echo "UA=$u $(env $E timeout 300 python scripts/bench_configs.py --configs 4 2>/dev/null | python -c 'import json,sys; print(" ".join("%s:%.2f" % (d["alg"], d["us_per_inner_step"]) for d in map(json.loads, sys.stdin.read().strip().splitlines())))')"
done; done | tee gpurun_out/ua8.txt
