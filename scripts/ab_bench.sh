#!/bin/bash
# Alternating A/B runs of a command on one box with libduquad_{A,B}.so (scripts/ab_build.sh).
# Usage: scripts/ab_bench.sh ROUNDS "command printing one line"
ROOT=$(cd "$(dirname "$0")/.." && pwd)
cp "$ROOT/paper_1504_05708_b200/libduquad.so" /tmp/libduquad_keep.so
for i in $(seq 1 "$1"); do
  for v in A B; do
    cp "$ROOT/paper_1504_05708_b200/libduquad_$v.so" "$ROOT/paper_1504_05708_b200/libduquad.so"
    echo "$v $(bash -c "$2" 2>/dev/null | tail -1)"
  done
done
cp /tmp/libduquad_keep.so "$ROOT/paper_1504_05708_b200/libduquad.so"
