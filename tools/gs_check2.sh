cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gsort.py -x -q --timeout 300 2>&1 | tail -3
bash tools/ab_gs.sh "$@"
bash tools/gs_trace.sh 2>&1 | grep -v "^ *1[01][0-9] |"
