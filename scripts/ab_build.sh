#!/bin/bash
# Build the library at two git revisions into paper_1504_05708_b200/libduquad_{A,B}.so (A/B timing on
# one box: scripts/ab_bench.sh).  Usage: scripts/ab_build.sh REV_A REV_B  (extra nvcc flags per
# variant: NVCC_A / NVCC_B, e.g. experiment macros)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
for v in A B; do
  rev=$([ $v = A ] && echo "$1" || echo "$2")
  tmp=$(mktemp -d)
  git -C "$ROOT" archive "$rev" paper_1504_05708_b200 include | tar -x -C "$tmp"
  extra=$([ $v = A ] && echo "$NVCC_A" || echo "$NVCC_B")
  (cd "$tmp" && DUQUAD_NVCC_EXTRA="$extra" python -c "from paper_1504_05708_b200 import build as b; b.build()" >/dev/null)
  cp "$tmp/paper_1504_05708_b200/libduquad.so" "$ROOT/paper_1504_05708_b200/libduquad_$v.so"
  rm -rf "$tmp"
done
ls -la "$ROOT"/paper_1504_05708_b200/libduquad_*.so
