# Q/G CTA split and Q row-step cost sweep for the byte-floor stream (config 2), default runs interleaved
set -x
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu"
for v in "" "DUQUAD_FUSED_NQ=70" "DUQUAD_FUSED_NQ=74" "" "DUQUAD_FUSED_NQ=62" "DUQUAD_FUSED_ROWCOST=16384" "" "DUQUAD_FUSED_ROWCOST=24576" "DUQUAD_FUSED_NQ=70 DUQUAD_FUSED_ROWCOST=16384" ""; do
  echo "[$v] $(env $v $B 2>/dev/null | python scripts/bench_brief.py)" >> gpurun_out/nq_sweep2.txt
done
cat gpurun_out/nq_sweep2.txt
