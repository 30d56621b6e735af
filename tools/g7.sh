cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 300 ./build/store_bench > gpurun_out/store_bench.txt 2>&1
timeout 600 python tools/e2e_probe.py cfg2 > gpurun_out/e2e_probe3.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_shard_gpu.py -q -x -k "pipelined or two_ranks" --timeout 600 > gpurun_out/pytest_g7.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g7.log
cat gpurun_out/store_bench.txt; tail -8 gpurun_out/e2e_probe3.txt; tail -3 gpurun_out/pytest_g7.log
