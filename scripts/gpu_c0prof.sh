# Full ncu capture (with source) of the config-0 whole-solve kernel
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_small_solve -c 1 -o gpurun_out/c0_small python scripts/bench_configs.py --configs 0 > gpurun_out/ncu_c0.log 2>&1; echo "ncu c0 rc=$?"
