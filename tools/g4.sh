cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 600 python tools/e2e_probe.py cfg2 > gpurun_out/e2e_probe2.txt 2>&1
timeout 600 python tools/e2e_probe.py cfg5 > gpurun_out/e2e_probe5.txt 2>&1
timeout 1500 python -m pytest tests/test_tntz_shim.py tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x -k "shim or pipelined or cfg4 or cfg5 or right_step or tall_thin" --timeout 1200 > gpurun_out/pytest_g4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g4.log
tail -15 gpurun_out/pytest_g4.log; cat gpurun_out/e2e_probe2.txt gpurun_out/e2e_probe5.txt
