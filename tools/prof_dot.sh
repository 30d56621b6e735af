#!/bin/bash
# ncu --set full of the rank-16 dot / norm kernel at cfg4 (one gpurun call):
# bash tools/prof_dot.sh  ->  gpurun_out/prof/{dot,norm}.ncu-rep
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out/prof
O=gpurun_out/prof
for op in ${1:-dot norm}; do
  D="python bench.py --op $op --steps 1 --warmup 3 --no-cpu"
  timeout 600 $D > $O/p_$op.log 2>&1 && \
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$op.csv $D > /dev/null 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:dot_r16 -s 1 -c 1 -o $O/$op $D > $O/ncu_$op.log 2>&1
  tail -1 $O/p_$op.log | cut -c1-300
done
ls -la $O
