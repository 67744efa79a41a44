set -x
mkdir -p gpurun_out
PROF_RHO=0 timeout 300 python scripts/prof_fused.py > gpurun_out/pf0.log 2>&1 && \
PROF_RHO=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_stream -s 1 -c 1 -o gpurun_out/prof_q4 python scripts/prof_fused.py > gpurun_out/ncu_q.log 2>&1; echo "ncu q rc=$?"
