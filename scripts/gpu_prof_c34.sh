set -x
mkdir -p gpurun_out
timeout 300 python scripts/dgemm_peak.py > gpurun_out/dgemm_peak.json 2>&1; cat gpurun_out/dgemm_peak.json
PROF_CFG=3 timeout 300 python scripts/prof_c34.py > gpurun_out/pc3.log 2>&1 && \
PROF_CFG=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batched -s 6 -c 2 -o gpurun_out/prof_c3 python scripts/prof_c34.py > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
PROF_CFG=4 timeout 600 python scripts/prof_c34.py > gpurun_out/pc4.log 2>&1 && \
PROF_CFG=4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass_._csr -s 6 -c 2 -o gpurun_out/prof_c4 python scripts/prof_c34.py > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
