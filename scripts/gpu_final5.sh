# Final checkpoint of the round, after the K4 block sizing and the dense-pass staging change: full GPU tests, smoke, default bench, per-config
# bench, reference arm, ncu launch list of the bench command and a full capture of config 1's passes
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python scripts/bench_brief.py < gpurun_out/bench.json
timeout 900 python scripts/bench_configs.py --configs 0,1,3,4 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"
CMD="python bench.py --steps 1 --warmup 0 --outer 2 --inner 5 --no-e2e --no-cpu"
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass_ -s 40 -c 2 -o gpurun_out/c1_pass python scripts/bench_configs.py --configs 1 --cases 1 > gpurun_out/ncu_c1.log 2>&1; echo "ncu c1 rc=$?"
