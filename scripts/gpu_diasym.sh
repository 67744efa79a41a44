# Symmetric half-band DIA (config 4): GPU tests of the CSR / sharded paths, then an A/B of the
# config-4 step with DUQUAD_DIA_SYM=0 (full band) / 1 (half band), alternated on one box
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_csr.py tests/test_gpu_sharded.py tests/test_gpu_state.py tests/test_gpu_eps.py -m gpu -x -q > gpurun_out/pytest_csr.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_csr.log
for i in 1 2; do
  for v in 0 1; do
    echo "SYM=$v $(DUQUAD_DIA_SYM=$v timeout 300 python scripts/bench_configs.py --configs 4 --cases 1 2>/dev/null | tail -1 | cut -c1-330)"
  done
done | tee gpurun_out/ab_diasym.txt
