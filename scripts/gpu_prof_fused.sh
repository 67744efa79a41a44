# GPU-box script: ncu --set full captures of k_fused_stream (rho = 0 Q-only, and rho = 1 default split)
set -x
mkdir -p gpurun_out
PROF_RHO=0 timeout 300 python scripts/prof_fused.py > gpurun_out/pf0.log 2>&1 && \
PROF_RHO=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_stream -s 1 -c 1 -o gpurun_out/prof_q python scripts/prof_fused.py > gpurun_out/ncu_q.log 2>&1; echo "ncu q rc=$?"
PROF_RHO=1 timeout 300 python scripts/prof_fused.py > gpurun_out/pf1.log 2>&1 && \
PROF_RHO=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_stream -s 1 -c 1 -o gpurun_out/prof_g python scripts/prof_fused.py > gpurun_out/ncu_g.log 2>&1; echo "ncu g rc=$?"
tail -3 gpurun_out/ncu_q.log gpurun_out/ncu_g.log
