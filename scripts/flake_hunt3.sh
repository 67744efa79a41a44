# full GPU suite twice, then the "csr or sharded" selection three times (no -x: every failure listed)
for i in 1 2; do
  echo "full $i: $(python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | grep -E '^FAILED|passed|failed' | tr '\n' ' ')"
done
for i in 1 2 3; do
  echo "sel $i: $(python -m pytest tests -m gpu -q -k 'csr or sharded or warm' -p no:cacheprovider 2>&1 | grep -E '^FAILED|passed|failed' | tr '\n' ' ')"
done
