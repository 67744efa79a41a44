# GPU-box script: byte-floor kernel parity tests + role-split sweep.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -15
timeout 600 python scripts/fused_sweep.py ${NQS:-0,60,68,74,80,88} > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?"
cat gpurun_out/sweep.jsonl; tail -5 gpurun_out/sweep.err
