set -x
mkdir -p gpurun_out
timeout 600 python scripts/sparse_sweep.py > gpurun_out/sparse_sweep.jsonl 2> gpurun_out/sparse_sweep.err; cat gpurun_out/sparse_sweep.jsonl; tail -3 gpurun_out/sparse_sweep.err
timeout 300 python scripts/prof_c4.py > gpurun_out/pc4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass_ -s 2 -c 4 -o gpurun_out/prof_c4_r2 python scripts/prof_c4.py > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_c4.log
