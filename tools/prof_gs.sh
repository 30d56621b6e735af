#!/bin/bash
# ncu --set full capture of the global-sort compute kernel (cfg2 or cfg5) + per-line stalls
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
C=${1:-cfg2}
O=gpurun_out/prof
mkdir -p $O
P="python tools/bench_entries.py --one $C"
timeout 300 $P > $O/gs_$C.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_gs_$C.csv $P > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:entries_gsort_kernel" -s 2 -c 1 -o $O/gs_$C $P > $O/ncu_gs_$C.log 2>&1
python tools/ncu_lines.py $O/gs_$C.ncu-rep 45 > $O/gs_${C}_lines.txt 2>&1
python tools/ncu_summary.py $O/gs_$C.ncu-rep > $O/gs_${C}_summary.txt 2>&1
tail -5 $O/ncu_gs_$C.log; head -60 $O/gs_${C}_lines.txt
