# ncu captures of the round-2 kernels: config 4 lane kernels, config 3 paired batched kernels
set -x
mkdir -p gpurun_out
timeout 300 python scripts/prof_c4.py > gpurun_out/pc4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:k_pass_ -s 2 -c 2 -o gpurun_out/prof_c4_r2final python scripts/prof_c4.py > gpurun_out/ncu_c4f.log 2>&1; echo "ncu c4 rc=$?"
PROF_CFG=3 timeout 300 python scripts/prof_c34.py > gpurun_out/pc3.log 2>&1 && \
PROF_CFG=3 timeout 900 ncu --set full --clock-control none -k regex:k_batched -s 2 -c 2 -o gpurun_out/prof_c3_r2final python scripts/prof_c34.py > gpurun_out/ncu_c3f.log 2>&1; echo "ncu c3 rc=$?"
