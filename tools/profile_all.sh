#!/bin/bash
# One gpurun call that regenerates every profile the docs cite:
#   bench lines (entries cfg2 with secondaries, entries cfg5, full, dot),
#   the ncu launch list of the headline bench command, and `ncu --set full`
#   captures of the dominant kernels.  Each ncu command runs only after the
#   same command exited 0 without ncu.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3"
timeout 900 $B > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --op entries5 --no-secondary --no-cpu --steps 3 --warmup 3 > gpurun_out/bench5.json 2>> gpurun_out/bench.err
P="python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu"
timeout 300 $P > gpurun_out/p.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_cfg2.csv $P > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:entries_compute -s 2 -c 1 \
    -o gpurun_out/prof_cfg2 $P > gpurun_out/ncu_cfg2.log 2>&1
P5="python tools/bench_entries.py --one cfg5"
timeout 300 $P5 > gpurun_out/p5.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_cfg5.csv $P5 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:entries_stream -s 1 -c 1 \
    -o gpurun_out/prof_cfg5 $P5 > gpurun_out/ncu_cfg5.log 2>&1
if [ -n "$FULLDOT" ]; then
F="python tools/prof_full.py 32"
timeout 300 $F > gpurun_out/pf.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_full.csv $F > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:full_tc -s 1 -c 1 \
    -o gpurun_out/prof_full $F > gpurun_out/ncu_full.log 2>&1
D="python bench.py --op dot --steps 1 --warmup 3"
timeout 300 $D > gpurun_out/pd.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_dot.csv $D > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:dot -s 1 -c 1 \
    -o gpurun_out/prof_dot $D > gpurun_out/ncu_dot.log 2>&1
fi
ls gpurun_out
