set -x
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -25
timeout 600 python bench.py --steps 2 --warmup 1 --outer 10 --inner 20 --no-e2e --no-cpu 2>&1 | tail -2
