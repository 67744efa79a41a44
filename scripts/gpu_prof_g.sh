set -x
mkdir -p gpurun_out
DUQUAD_FUSED_NQ=${NQ:-60} PROF_RHO=1 timeout 300 python scripts/prof_fused.py > gpurun_out/pf1.log 2>&1 && \
DUQUAD_FUSED_NQ=${NQ:-60} PROF_RHO=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_stream -s 1 -c 1 -o gpurun_out/prof_g6 python scripts/prof_fused.py > gpurun_out/ncu_g.log 2>&1; echo "ncu g rc=$?"
