#!/bin/bash
# A/B of kernel build variants on cfg2 / cfg5: bash tools/ab_variants.sh v1 v2 ...
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
for i in 1 2; do
  for c in cfg2 cfg5; do
    echo "base $c $(python tools/bench_entries.py --one $c | cut -c1-220)"
    for v in "$@"; do echo "$v $c $(TNB_LIB=build/variants/$v/libtnb.so python tools/bench_entries.py --one $c | cut -c1-220)"; done
  done
done
