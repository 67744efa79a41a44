# GPU-box script: batched (config 3) parity tests, per-config timing and one ncu capture of both passes.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "batch or mpc or warm" > gpurun_out/pytest_c3.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_c3.log
timeout 600 python scripts/bench_configs.py --configs 3 > gpurun_out/c3.jsonl 2> gpurun_out/c3.err; echo "bench rc=$?"
cat gpurun_out/c3.jsonl; tail -3 gpurun_out/c3.err
if [ -n "$DO_NCU" ]; then
PROF_CFG=3 timeout 300 python scripts/prof_c34.py > gpurun_out/pc3.log 2>&1 && \
PROF_CFG=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batched -s 6 -c 2 -o gpurun_out/prof_c3 python scripts/prof_c34.py > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
fi
