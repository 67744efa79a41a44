# Q-role piece cut: diagonal-tile step weight (DUQUAD_FUSED_DIAG) x Q/G split (DUQUAD_FUSED_NQ)
mkdir -p gpurun_out
cp paper_1504_05708_b200/libduquad.so /tmp/keep.so
cp paper_1504_05708_b200/libduquad_T.so paper_1504_05708_b200/libduquad.so
for cfg in "1.15 66" "1.15 70" "1.3 70"; do set -- $cfg; DUQUAD_FUSED_DIAG=$1 DUQUAD_FUSED_NQ=$2 timeout 300 python scripts/role_trace.py 2>&1 | tail -1 | sed "s/^/DIAG=$1 /"; done | tee gpurun_out/role_trace3.jsonl | cut -c1-200
cp /tmp/keep.so paper_1504_05708_b200/libduquad.so
for i in 1 2; do
  for cfg in "1.0 70" "1.12 66" "1.12 68" "1.12 70" "1.2 68" "1.2 70" "1.2 72"; do
    set -- $cfg
    echo "DIAG=$1 NQ=$2 $(DUQUAD_FUSED_DIAG=$1 DUQUAD_FUSED_NQ=$2 timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python scripts/bench_brief.py)"
  done
done | tee gpurun_out/diag_sweep.txt
