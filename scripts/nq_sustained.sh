# GPU-box script: the byte-floor Q/G CTA split under sustained (power-capped) load -- bench.py
# runs with DUQUAD_FUSED_NQ overridden, interleaved with the default split to separate the split's
# effect from the box's clock drift.  One JSON summary line per run.
mkdir -p gpurun_out
for nq in 0 58 0 74 0 62 0 70; do
  if [ "$nq" = 0 ]; then unset DUQUAD_FUSED_NQ; else export DUQUAD_FUSED_NQ=$nq; fi
  timeout 400 python bench.py --no-cpu --no-e2e --steps 2 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'nq': $nq, 'value': d['value'], 'ms_launch': d['roofline']['ms_per_launch'], 'sm_mhz': d['clocks']['sm_mhz']}))"
done
