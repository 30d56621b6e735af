#!/bin/bash
# full() at cfg3 across libtnb build variants: bash tools/ab_full_variants.sh v1 v2 ...
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
for i in 1 2; do
for v in base "$@"; do
  echo "== $v"
  if [ $v = base ]; then unset TNB_LIB; else export TNB_LIB=build/variants/$v/libtnb.so; fi
  python bench.py --op full --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ms/step', d['ms_per_step'], 'gemm ms', d['roofline'].get('kernel_ms'), 'GB/s', d['value'])"
done
done
