# A/B of the lane kernels' register cap (DQ_LANE_MINB) on config 4
set -x
mkdir -p gpurun_out
for MB in 1 6 8; do
DUQUAD_NVCC_EXTRA="-DDQ_LANE_MINB=$MB" python -c "from paper_1504_05708_b200 import build as b; b.build()" && \
timeout 300 python scripts/sparse_sweep.py 2>/dev/null | head -1 | sed "s/^/minb=$MB /" >> gpurun_out/minb.txt
done
cat gpurun_out/minb.txt
