mkdir -p gpurun_out
E2E_OUTER=10 timeout 600 python scripts/e2e_phases.py 2>&1 | tail -3 | tee gpurun_out/e2e_phases.txt
