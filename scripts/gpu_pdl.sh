# A/B of programmatic dependent launch (DUQUAD_PDL) and the dense passes' pre-wait row prefetch
# (DQ_PDL_PF) on configs 1, 4 (bench_configs) and 2 (bench.py)
set -x
mkdir -p gpurun_out
for PF in 1 0; do
DUQUAD_NVCC_EXTRA="-DDQ_PDL_PF=$PF" python -c "from paper_1504_05708_b200 import build as b; b.build()" || exit 1
for P in 1 0; do
DUQUAD_PDL=$P timeout 600 python scripts/bench_configs.py --configs 0,1,3,4 --cases 2 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(json.dumps(dict(pf=$PF, pdl=$P, cfg=d['config'], alg=d['alg'], rho=d['rho'], us=d['us_per_inner_step'])))" >> gpurun_out/pdl_ab.jsonl
done; done
python -c "from paper_1504_05708_b200 import build as b; b.build()"
for P in 1 0; do
DUQUAD_PDL=$P timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(dict(pdl=$P, value=d['value'], frac=d['roofline']['frac'], clocks=d.get('clocks'))))" >> gpurun_out/pdl_ab.jsonl
done
cat gpurun_out/pdl_ab.jsonl
