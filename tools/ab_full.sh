#!/bin/bash
# full() at cfg3 with / without the lockstep tile order: bash tools/ab_full.sh
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
for i in 1 2; do
for v in 1 0; do
  echo "== TNB_FULL_LOCKSTEP=$v"
  TNB_FULL_LOCKSTEP=$v python bench.py --op full --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ms/step', d['ms_per_step'], 'gemm ms', d['roofline'].get('kernel_ms'), 'GB/s', d['value'], d.get('parity'))"
done
done
