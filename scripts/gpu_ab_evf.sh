# A/B: byte-floor matrix stream without (A) / with (B) the L2 evict-first policy (DQ_STREAM_EVF)
mkdir -p gpurun_out
bash scripts/ab_bench.sh 3 "timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu | python scripts/bench_brief.py" | tee gpurun_out/ab_evf.txt
