# PDL on/off (DUQUAD_PDL=2 / 0) on configs 0, 1 (bench_configs) and 2 (bench.py)
set -x
mkdir -p gpurun_out
for P in 2 0; do
DUQUAD_PDL=$P timeout 600 python scripts/bench_configs.py --configs 0,1 --cases 4 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(json.dumps(dict(pdl=$P, cfg=d['config'], alg=d['alg'], rho=d['rho'], us=d['us_per_inner_step'])))" >> gpurun_out/pdl2.jsonl
DUQUAD_PDL=$P timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(dict(pdl=$P, value=d['value'], frac=d['roofline']['frac'], epi=d['roofline']['epilogue']['ms_per_launch'], clocks=d.get('clocks'))))" >> gpurun_out/pdl2.jsonl
done
cat gpurun_out/pdl2.jsonl
