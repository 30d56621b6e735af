#!/bin/bash
# launch list + ncu --set full of the whole-call cfg3 full() GEMM (one gpurun call):
# bash tools/prof_full.sh  ->  gpurun_out/prof/full.ncu-rep, launches_full.csv
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out/prof
O=gpurun_out/prof
F="python tools/prof_full.py 256"
timeout 300 $F > $O/p_full.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_full.csv $F > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:full_tc_gemm -s 1 -c 1 -o $O/full $F > $O/ncu_full.log 2>&1
cat $O/p_full.log; ls -la $O | grep full
