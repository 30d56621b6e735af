#!/bin/bash
# A/B of global-sort build variants: bash tools/ab_gs.sh v1 v2 ...
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
for c in cfg2 cfg5; do
  echo "base $c $(python tools/bench_entries.py --one $c | cut -c1-260)"
  for v in "$@"; do echo "$v $c $(TNB_LIB=build/variants/$v/libtnb.so python tools/bench_entries.py --one $c | cut -c1-260)"; done
done
