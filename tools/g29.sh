cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
for i in 1 2; do
python bench.py --op full --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('base', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3))"
TNB_LIB=build/variants/epi8/libtnb.so python bench.py --op full --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('epi8', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3))"
done
TNB_LIB=build/variants/epi8/libtnb.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_guards.py -q -x -k "full or cfg3" --timeout 600 2>&1 | tail -2
