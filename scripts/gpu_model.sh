# Q piece cut: fitted diagonal-step model (default) vs the flat 1.12 weight, x Q/G split
mkdir -p gpurun_out
for i in 1 2; do
  for cfg in "flat 66" "fit 66" "fit 64" "fit 68"; do
    set -- $cfg
    if [ $1 = flat ]; then E="DUQUAD_FUSED_DIAG=1.12 DUQUAD_FUSED_DSLOPE=0"; else E=""; fi
    echo "$1 NQ=$2 $(env $E DUQUAD_FUSED_NQ=$2 timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python scripts/bench_brief.py)"
  done
done | tee gpurun_out/model_sweep.txt
