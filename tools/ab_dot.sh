#!/bin/bash
# A/B of libtnb build variants on cfg4 dot / norm: bash tools/ab_dot.sh v1 v2 ...
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
for v in base "$@" base; do
  echo "== $v"
  if [ $v = base ]; then python tools/bench_dot.py; else TNB_LIB=build/variants/$v/libtnb.so python tools/bench_dot.py; fi
done
