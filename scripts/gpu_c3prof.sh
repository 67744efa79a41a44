set -x
mkdir -p gpurun_out
PROF_CFG=3 timeout 300 python scripts/prof_c34.py > gpurun_out/pc3.log 2>&1 && \
PROF_CFG=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batched -s 2 -c 2 -o gpurun_out/prof_c3_r2 python scripts/prof_c34.py > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"; tail -2 gpurun_out/ncu_c3.log
