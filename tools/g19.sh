cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
for i in 1 2; do
python tools/bench_entries.py --one cfg2 > gpurun_out/ab_l1pf_on_$i.txt 2>&1
TNB_LIB=build/variants/nol1pf/libtnb.so python tools/bench_entries.py --one cfg2 > gpurun_out/ab_l1pf_off_$i.txt 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "cfg2 or r32 or bucketed_tiles or merging" --timeout 600 > gpurun_out/pytest_g19.log 2>&1; tail -2 gpurun_out/pytest_g19.log
for f in gpurun_out/ab_l1pf_*; do echo $f; cut -c1-200 $f; done
