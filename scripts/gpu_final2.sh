# End-of-round-2 checkpoint: full GPU tests + smoke, default bench, per-config bench, ncu launch list of
# the bench command, full ncu captures of the config-2 stream kernel and the config-4 pass-A kernel
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python scripts/bench_brief.py < gpurun_out/bench.json
timeout 900 python scripts/bench_configs.py --configs 0,1,3,4 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
CMD="python bench.py --steps 1 --warmup 0 --outer 2 --inner 5 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_stream -s 3 -c 1 -o gpurun_out/prof_c2_r2final $CMD > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
timeout 300 python scripts/prof_c4.py > gpurun_out/pc4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:k_pass_ -s 2 -c 2 -o gpurun_out/prof_c4_r2sym python scripts/prof_c4.py > gpurun_out/ncu_c4f.log 2>&1; echo "ncu c4 rc=$?"
