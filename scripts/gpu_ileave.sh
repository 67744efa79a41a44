# A/B: G rows to the pairs in contiguous blocks (A) / round robin (B, DQ_G_INTERLEAVE=1); B's fused tests first
mkdir -p gpurun_out
cp paper_1504_05708_b200/libduquad.so /tmp/keep.so
cp paper_1504_05708_b200/libduquad_B.so paper_1504_05708_b200/libduquad.so
timeout 900 python -m pytest tests/test_gpu_fused.py -m gpu -x -q > gpurun_out/pytest_il.log 2>&1; echo "pytest(B) rc=$?"; tail -2 gpurun_out/pytest_il.log
cp /tmp/keep.so paper_1504_05708_b200/libduquad.so
bash scripts/ab_bench.sh 3 "timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu | python scripts/bench_brief.py" | tee gpurun_out/ab_ileave.txt
