# Byte-floor stream, instrumentation build (DQ_TRACE_G): where the G role's time goes
mkdir -p gpurun_out
cp paper_1504_05708_b200/libduquad_B.so paper_1504_05708_b200/libduquad.so
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/trace_g.log 2>&1; echo "rc=$?"
grep TRACE_G gpurun_out/trace_g.log | tail -4
tail -1 gpurun_out/trace_g.log | python scripts/bench_brief.py
