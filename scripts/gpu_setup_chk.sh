# Setup changes (G' from the uploaded G rows; device finiteness check of host Q / G): parity and
# batched tests, then the end-to-end phase times
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py tests/test_gpu_eq_h.py tests/test_gpu_warm.py -m gpu -x -q > gpurun_out/pytest_setup.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_setup.log
E2E_OUTER=10 timeout 600 python scripts/e2e_phases.py 2>&1 | tail -3 | tee gpurun_out/e2e_phases2.txt
