cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; lscpu >> gpurun_out/host.txt 2>&1; free -g >> gpurun_out/host.txt
timeout 600 python tools/e2e_probe.py cfg2 > gpurun_out/e2e_probe.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m "gpu and not slow" -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log gpurun_out/e2e_probe.txt; head -3 gpurun_out/host.txt
