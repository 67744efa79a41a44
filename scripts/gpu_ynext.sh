# A/B: Q-role y window loaded on use (A, DQ_YNEXT=0) / one window ahead (B, default); fused GPU tests first
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_sharded.py -m gpu -x -q > gpurun_out/pytest_yn.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_yn.log
bash scripts/ab_bench.sh 3 "timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu | python scripts/bench_brief.py" | tee gpurun_out/ab_ynext.txt
for nq in 64 68; do echo "B NQ=$nq $(DUQUAD_FUSED_NQ=$nq timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python scripts/bench_brief.py)"; done | tee -a gpurun_out/ab_ynext.txt
