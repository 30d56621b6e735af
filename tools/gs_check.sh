cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gsort.py -x -q --timeout 300 > gpurun_out/gs_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gs_tests.log
tail -30 gpurun_out/gs_tests.log
for c in cfg2 cfg5; do
  timeout 300 python tools/bench_entries.py --one $c --algo 0 > gpurun_out/gs_$c.json 2> gpurun_out/gs_$c.err; echo "rc=$?"; cat gpurun_out/gs_$c.json; tail -3 gpurun_out/gs_$c.err
  TNB_ENTRIES_GSORT=0 timeout 300 python tools/bench_entries.py --one $c --algo 0
done
