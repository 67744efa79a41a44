# Byte-floor stream: per-CTA durations of one launch (DQ_TRACE_ROLE build), then a Q/G split sweep
mkdir -p gpurun_out
cp paper_1504_05708_b200/libduquad.so /tmp/keep.so
cp paper_1504_05708_b200/libduquad_T.so paper_1504_05708_b200/libduquad.so
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/trace_role.log 2>&1; echo "rc=$?"
cp /tmp/keep.so paper_1504_05708_b200/libduquad.so
grep TRACE_ROLE gpurun_out/trace_role.log | head -24
for i in 1 2; do
  for nq in 66 62 70; do
    echo "NQ=$nq $(DUQUAD_FUSED_NQ=$nq timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python scripts/bench_brief.py)"
  done
done | tee gpurun_out/nq_sweep3.txt
