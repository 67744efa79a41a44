# Three-way alternating A/B/C of the default bench (libduquad_{A,B,C}.so), after the fused GPU tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_sharded.py tests/test_gpu_nccl_self.py -m gpu -x -q > gpurun_out/pytest_ab3.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ab3.log
ROOT=$(pwd)
cp paper_1504_05708_b200/libduquad.so /tmp/keep.so
for i in 1 2 3; do
  for v in A B C; do
    cp paper_1504_05708_b200/libduquad_$v.so paper_1504_05708_b200/libduquad.so
    echo "$v $(timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu 2>gpurun_out/ab3_$v.err | python scripts/bench_brief.py)"
  done
done | tee gpurun_out/ab3.txt
cp /tmp/keep.so paper_1504_05708_b200/libduquad.so
