cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f64.py -q -x -k "rank_general or two_table or golden or merging or f64" --timeout 600 > gpurun_out/pytest_g12.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g12.log
timeout 900 python tools/generic_probe.py > gpurun_out/generic_probe3.txt 2>&1
tail -15 gpurun_out/pytest_g12.log; cat gpurun_out/generic_probe3.txt
