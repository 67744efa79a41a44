# Byte-floor stream: per-CTA start/end of one launch (DQ_TRACE_ROLE build, scripts/role_trace.py)
# at two Q/G splits, then a Q/G split sweep of the production build
mkdir -p gpurun_out
cp paper_1504_05708_b200/libduquad.so /tmp/keep.so
cp paper_1504_05708_b200/libduquad_T.so paper_1504_05708_b200/libduquad.so
for nq in 66 70 74; do DUQUAD_FUSED_NQ=$nq timeout 300 python scripts/role_trace.py 2>&1 | tail -1; done | tee gpurun_out/role_trace.jsonl | cut -c1-200
cp /tmp/keep.so paper_1504_05708_b200/libduquad.so
for i in 1 2; do
  for nq in 66 70 72 74 76; do
    echo "NQ=$nq $(DUQUAD_FUSED_NQ=$nq timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python scripts/bench_brief.py)"
  done
done | tee gpurun_out/nq_sweep4.txt
