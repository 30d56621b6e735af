#!/bin/bash
# ncu evidence for the cfg2 plan alternative with L2-resident tables (P012 /
# S789, 4 MB each, 4 sorted modes): DRAM bytes per launch vs the planner's
# P0123 / S6789 (128 MB each, 2 sorted modes).
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out/prof
export TNB_PREFIX_MAX_ROWS=32768 TNB_SUFFIX_MAX_ROWS=32768
P="python tools/bench_entries.py --one cfg2"
timeout 300 $P > gpurun_out/prof/l2plan_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:entries_compute_kernel<.*\(bool\)0>" -s 1 -c 1 \
    -o gpurun_out/prof/cfg2_l2plan $P > gpurun_out/prof/ncu_l2plan.log 2>&1
tail -2 gpurun_out/prof/ncu_l2plan.log; cat gpurun_out/prof/l2plan_plain.log | cut -c1-300
