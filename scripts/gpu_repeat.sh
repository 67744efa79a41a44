# Run-to-run spread of the headline: the default bench three times back to back on one box
set -x
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 600 python bench.py --no-cpu > gpurun_out/repeat_$i.json 2> gpurun_out/repeat_$i.err; echo "bench $i rc=$?"; python scripts/bench_brief.py < gpurun_out/repeat_$i.json
done
