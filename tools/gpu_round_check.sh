cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; echo "bench rc=$?" >> gpurun_out/bench_r02b.err
timeout 1800 python -m pytest tests -q -m "gpu and not slow" --timeout 1200 > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke2.log
tail -4 gpurun_out/pytest_full.log; tail -2 gpurun_out/smoke2.log; tail -3 gpurun_out/bench_r02b.err
