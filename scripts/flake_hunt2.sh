# the "csr or sharded" GPU test selection repeated (it failed intermittently), PDL default vs off
for P in 1 0; do
  for i in 1 2 3; do
    echo "PDL=$P run $i: $(DUQUAD_PDL=$P python -m pytest tests -m gpu -q -x -k 'csr or sharded' -p no:cacheprovider 2>&1 | grep -E 'passed|FAILED' | tr '\n' ' ')"
  done
done
