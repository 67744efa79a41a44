# Config 3 group-width sweep (env overrides read once per process): pass A (paired) NT, pass B NT
set -x
mkdir -p gpurun_out
for A in 7 5 4; do for B in 4 3 7; do
DUQUAD_NTA_PAIR=$A DUQUAD_NTB=$B timeout 300 python scripts/bench_configs.py --configs 3 --reps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(dict(nta=$A, ntb=$B, us=d['us_per_inner_step'], a=d['ms_pass_a']*1e3, b=d['ms_pass_b']*1e3)))" >> gpurun_out/batched_sweep.jsonl
done; done
cat gpurun_out/batched_sweep.jsonl
