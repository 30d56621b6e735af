cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_guards.py -q -x --timeout 600 > gpurun_out/pytest_guards.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_guards.log
timeout 900 python tools/generic_probe.py > gpurun_out/generic_probe.txt 2>&1
tail -5 gpurun_out/pytest_guards.log; cat gpurun_out/generic_probe.txt
