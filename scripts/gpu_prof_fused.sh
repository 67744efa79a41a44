python scripts/prof_fused.py > gpurun_out/pf.log 2>&1 && \
DUQUAD_FUSED_NQ=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused_stream -s 1 -c 1 -o gpurun_out/prof_fusedg python scripts/prof_fused.py > gpurun_out/ncu_fg.log 2>&1; echo "rc=$?"
DUQUAD_FUSED_NQ=148 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused_stream -s 1 -c 1 -o gpurun_out/prof_fusedq python scripts/prof_fused.py > gpurun_out/ncu_fq.log 2>&1; echo "rc=$?"
