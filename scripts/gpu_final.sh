# GPU-box script: full GPU tests, smoke, per-config timings (0,1,3,4), ncu captures of the batched passes.
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 900 python scripts/bench_configs.py --configs 0,1,3,4 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
cat gpurun_out/configs.jsonl
if [ -n "$DO_NCU" ]; then
PROF_CFG=3 timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_batched$' -s 0 -c 2 -o gpurun_out/prof_c3 python scripts/prof_c34.py > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
fi
