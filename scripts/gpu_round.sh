# GPU-box script: full GPU tests, smoke, default bench, ncu launch list of the bench command and
# one --set full capture of the dominant kernel (k_fused_stream).  Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [ -z "$SKIP_TESTS" ]; then
timeout 1800 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
fi
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
if [ -n "$DO_NCU" ]; then
NCUCMD="python bench.py --steps 1 --warmup 0 --outer 2 --inner 5 --no-e2e --no-cpu"
timeout 600 $NCUCMD > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $NCUCMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 2 -o gpurun_out/prof_round $NCUCMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
fi
ls gpurun_out
