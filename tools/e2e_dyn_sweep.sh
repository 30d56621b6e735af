#!/bin/bash
# the self-balancing host pipeline against the static raw fraction on cfg2: bash tools/e2e_dyn_sweep.sh
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
for env in "" "TNB_E2E_THREADS=12" "TNB_E2E_THREADS=8" "TNB_E2E_CHUNK_LOG2=19" "TNB_E2E_DYNAMIC=0" "TNB_E2E_RAW_FRAC=0.5"; do
  echo "== $env"
  env $env python tools/e2e_dyn.py
done
