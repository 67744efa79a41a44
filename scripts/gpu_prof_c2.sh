# one full ncu capture (with source) of the byte-floor stream kernel on a short config-2 solve
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --outer 2 --inner 5 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/plain_c2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_stream -s 3 -c 1 -o gpurun_out/prof_c2_r2 $CMD > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_c2.log
