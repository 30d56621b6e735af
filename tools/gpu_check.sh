#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, then (only if the plain runs exited
# 0) an ncu launch list and full captures of the entries and full() kernels.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
TESTSEL=${TESTSEL:-"gpu and not slow"}
if [ -z "$SKIP_TESTS" ]; then
timeout 1200 python -m pytest tests -q -m "$TESTSEL" --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
fi
timeout 900 python bench.py ${BENCH_ARGS:---steps 5 --warmup 3} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
if [ -n "$NCU" ]; then
  P="python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu"
  timeout 300 $P > gpurun_out/ncu_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_launch.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_K:-entries_compute} \
      -s 1 -c ${NCU_C:-1} -o gpurun_out/prof_entries $P > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_full.log
fi
if [ -n "$NCU_FULL" ]; then
  F="python tools/prof_full.py 32"
  timeout 300 $F > gpurun_out/prof_full_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:full_tc \
      -s 1 -c 1 -o gpurun_out/prof_full $F > gpurun_out/ncu_fullk.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_fullk.log
fi
tail -3 gpurun_out/pytest_gpu.log 2>/dev/null; cat gpurun_out/smoke.log 2>/dev/null; cut -c1-400 gpurun_out/bench.json; tail -3 gpurun_out/bench.err; cat gpurun_out/prof_full_plain.log 2>/dev/null
