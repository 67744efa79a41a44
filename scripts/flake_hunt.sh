# repeat the warm-start tests that failed intermittently, with PDL on and off
T="tests/test_gpu_sharded.py::test_sharded_byte_floor_ragged_warm_start_and_dual_average tests/test_gpu_warm.py::test_warm_start_csr tests/test_gpu_warm.py"
for P in 1 0; do
  f=0
  for i in $(seq 1 8); do
    DUQUAD_PDL=$P python -m pytest $T -q -p no:cacheprovider 2>&1 | tail -1 | grep -q failed && f=$((f+1))
  done
  echo "PDL=$P failures $f / 8"
done
