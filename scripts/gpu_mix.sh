# A/B: SELL pass A slices in storage order (A, DQ_SELL_MIX=0) / Q and G slices interleaved (B); CSR tests with B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_csr.py tests/test_gpu_sharded.py -m gpu -x -q > gpurun_out/pytest_mix.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_mix.log
bash scripts/ab_bench.sh 3 "timeout 300 python scripts/bench_configs.py --configs 4 --cases 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d[\"us_per_inner_step\"],2), round(1e3*d[\"ms_pass_a\"],1), round(1e3*d[\"ms_pass_b\"],1))'" | tee gpurun_out/ab_mix.txt
