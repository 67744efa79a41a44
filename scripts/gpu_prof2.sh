set -x
python scripts/dgemm_peak.py
C3="python scripts/bench_configs.py --configs 3 --reps 1 --cases 1"
C4="python scripts/bench_configs.py --configs 4 --reps 1 --cases 1"
$C3 > gpurun_out/c3.log 2>&1 && timeout 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:k_batched -s 2 -c 2 -o gpurun_out/prof_batched $C3 > gpurun_out/ncu_b.log 2>&1; echo "ncu b rc=$?"
$C4 > gpurun_out/c4.log 2>&1 && timeout 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:csr -s 2 -c 2 -o gpurun_out/prof_csr $C4 > gpurun_out/ncu_c.log 2>&1; echo "ncu c rc=$?"
