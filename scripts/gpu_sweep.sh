# GPU-box script: fused-kernel role-split sweep + one ncu --set full capture of k_fused_stream.
set -x
mkdir -p gpurun_out
timeout 900 python scripts/fused_sweep.py ${NQS:-0,2,40,60,74,90,110,148} > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?"
cat gpurun_out/sweep.jsonl; tail -3 gpurun_out/sweep.err
if [ -n "$DO_NCU" ]; then
timeout 300 python scripts/prof_fused.py > gpurun_out/pf.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_stream -s 1 -c 1 -o gpurun_out/prof_fused python scripts/prof_fused.py > gpurun_out/ncu_f.log 2>&1; echo "ncu rc=$?"
fi
