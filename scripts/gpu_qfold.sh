# q folded into pass A (CSR): CSR / sharded / state / eps / monitored tests, then config 4 with
# DUQUAD_QFOLD = 0 / 1 alternated
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_csr.py tests/test_gpu_sharded.py tests/test_gpu_state.py tests/test_gpu_eps.py tests/test_gpu_monitored.py tests/test_gpu_warm.py tests/test_gpu_nccl_self.py -m gpu -x -q > gpurun_out/pytest_qfold.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_qfold.log
for i in 1 2 3; do for f in 0 1; do
  echo "QFOLD=$f $(DUQUAD_QFOLD=$f timeout 300 python scripts/bench_configs.py --configs 4 --cases 1 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["us_per_inner_step"],2), round(1e3*d["ms_pass_a"],1), round(1e3*d["ms_pass_b"],1))')"
done; done | tee gpurun_out/qfold.txt
