cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 300 python tools/widen_probe.py > gpurun_out/widen_probe.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "full or cfg3 or cfg1" --timeout 600 > gpurun_out/pytest_g5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g5.log
for v in 1 0; do TNB_FULL_TMA_STORE=$v timeout 300 python bench.py --op full --steps 10 --warmup 3 > gpurun_out/full_tma$v.json 2>&1; done
tail -3 gpurun_out/pytest_g5.log; cat gpurun_out/widen_probe.txt; for v in 1 0; do python -c "
import json,sys; d=json.loads(open('gpurun_out/full_tma$v.json').read().strip().splitlines()[-1]); r=d['roofline']
print('tma=$v', round(d['ms_per_step'],3), 'ms', round(d['value'],1), 'GB/s kernel', round(r['kernel_ms'],3), 'frac', round(r['frac'],3), 'wo', round(r.get('frac_vs_write_only',0),3), d.get('parity_gate'))" || tail -5 gpurun_out/full_tma$v.json; done
