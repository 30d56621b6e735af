cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "batched or golden_entries" --timeout 600 > gpurun_out/pytest_g11.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g11.log
timeout 900 python tools/generic_probe.py > gpurun_out/generic_probe2.txt 2>&1
tail -5 gpurun_out/pytest_g11.log; cat gpurun_out/generic_probe2.txt
