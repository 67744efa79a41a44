# compute-sanitizer passes over the shipped library: memcheck / racecheck / synccheck on smoke()
# (K4 small kernel + the byte-floor stream and epilogue) and memcheck on the parity, CSR and batched
# GPU tests.  Logs under gpurun_out/; never a timing run.
set -x
mkdir -p gpurun_out
CS="compute-sanitizer --error-exitcode 9 --print-limit 20"
timeout 240 $CS --tool memcheck python __graft_entry__.py smoke > gpurun_out/san_memcheck_smoke.log 2>&1; echo "memcheck smoke rc=$?"; tail -2 gpurun_out/san_memcheck_smoke.log
timeout 300 $CS --tool racecheck python __graft_entry__.py smoke > gpurun_out/san_racecheck_smoke.log 2>&1; echo "racecheck smoke rc=$?"; tail -2 gpurun_out/san_racecheck_smoke.log
timeout 200 $CS --tool synccheck python __graft_entry__.py smoke > gpurun_out/san_synccheck_smoke.log 2>&1; echo "synccheck smoke rc=$?"; tail -2 gpurun_out/san_synccheck_smoke.log
timeout 600 $CS --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_csr.py tests/test_gpu_batched.py -m gpu -q > gpurun_out/san_memcheck_tests.log 2>&1; echo "memcheck tests rc=$?"; tail -4 gpurun_out/san_memcheck_tests.log
