cd "${GRAFT_REPO_ROOT:-$(pwd)}"
for i in 1 2; do for v in 1 0; do for c in cfg2 cfg5; do echo "tcgen05=$v $c $(TNB_TABLE_TCGEN05=$v python tools/bench_entries.py --one $c | cut -c1-230)"; done; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "bucketed or cfg2 or cfg5 or merging or wide or batched" --timeout 600 2>&1 | tail -2
