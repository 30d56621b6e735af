#!/bin/bash
# Launch list + `ncu --set full` capture of the global-sort compute kernel on the
# headline command (cfg2, bench.py), each ncu pass only after the same command
# exited 0 without ncu; per-line stalls and the prep / scatter kernels too.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out/prof
O=gpurun_out/prof
P2="python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu"
timeout 300 $P2 > $O/p2_gsort.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2_gsort.csv $P2 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:entries_gsort_kernel" -s 2 -c 1 -o $O/cfg2_gsort $P2 > $O/ncu_cfg2_gsort.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:gs_prep_kernel|gs_scatter_kernel" -s 4 -c 2 -o $O/cfg2_gsort_sort $P2 > $O/ncu_cfg2_gsort_sort.log 2>&1
python tools/ncu_lines.py $O/cfg2_gsort.ncu-rep 40 > $O/cfg2_gsort_lines.txt 2>&1
mkdir -p build/tools
[ -x build/tools/gather_bench ] || nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o build/tools/gather_bench tools/gather_bench.cu
build/tools/gather_bench 23 25 > $O/gather_bench_2p23.txt 2>&1
build/tools/gather_bench 20 24 > $O/gather_bench_2p20.txt 2>&1
tail -3 $O/p2_gsort.log | cut -c1-300; ls -la $O | tail -12
