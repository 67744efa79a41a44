# Config 4 after the symmetric DIA: SELL pass-A register cap (DQ_SELLA_MINB 4 / 5 / 6 builds) and the
# SELL load-round width (DUQUAD_LANE_UA 4 / 8), alternated on one box
mkdir -p gpurun_out
cp paper_1504_05708_b200/libduquad.so /tmp/keep.so
for i in 1 2; do
  for v in base M5 M6 UA8; do
    case $v in base|UA8) cp /tmp/keep.so paper_1504_05708_b200/libduquad.so;; *) cp paper_1504_05708_b200/libduquad_$v.so paper_1504_05708_b200/libduquad.so;; esac
    E=""; [ $v = UA8 ] && E="DUQUAD_LANE_UA=8"
    echo "$v $(env $E timeout 300 python scripts/bench_configs.py --configs 4 --cases 1 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["us_per_inner_step"],2), round(1e3*d["ms_pass_a"],1), round(1e3*d["ms_pass_b"],1))')"
  done
done | tee gpurun_out/c4_sweep.txt
cp /tmp/keep.so paper_1504_05708_b200/libduquad.so
# config 1 re-check (its two-pass / K3 kernels were not changed this session)
timeout 600 python scripts/bench_configs.py --configs 1 > gpurun_out/c1_recheck.jsonl 2>/dev/null; python -c "
import json
for l in open('gpurun_out/c1_recheck.jsonl'):
    d=json.loads(l); print('c1', d['alg'], d['rho'], round(d['us_per_inner_step'],2))"
