#!/bin/bash
# One gpurun call regenerating the round-2 profiles: launch lists and
# `ncu --set full` captures of the dominant kernels (each ncu command only
# after the same command exited 0 without ncu in this call).
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out/prof
O=gpurun_out/prof
P2="python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu"
timeout 300 $P2 > $O/p2.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv $P2 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:entries_compute_kernel<.*\(bool\)0>" -s 2 -c 1 -o $O/cfg2 $P2 > $O/ncu_cfg2.log 2>&1
P5="python tools/bench_entries.py --one cfg5"
timeout 300 $P5 > $O/p5.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv $P5 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:entries_stream_kernel<.*\(bool\)0>" -s 1 -c 1 -o $O/cfg5 $P5 > $O/ncu_cfg5.log 2>&1
for op in dot norm; do
  D="python bench.py --op $op --steps 1 --warmup 3 --no-cpu"
  timeout 600 $D > $O/p_$op.log 2>&1 && \
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$op.csv $D > /dev/null 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:dot_r16 -s 1 -c 1 -o $O/$op $D > $O/ncu_$op.log 2>&1
done
for w in two_table dot_chunk batched; do
  X="python tools/prof_extra.py $w"
  timeout 300 $X > $O/px_$w.log 2>&1 && \
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$w.csv $X > /dev/null 2>&1
done
X="python tools/prof_extra.py two_table"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:two_table -s 1 -c 1 -o $O/two_table $X > $O/ncu_tt.log 2>&1
X="python tools/prof_extra.py dot_chunk"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dot_mma -s 1 -c 1 -o $O/dot_mma $X > $O/ncu_dc.log 2>&1
ls -la $O
