cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
python tools/bench_entries.py --sweep cfg2 '{}' '{"TNB_PREFIX_MAX_ROWS":"32768"}' '{"TNB_SUFFIX_MAX_ROWS":"32768"}' '{"TNB_PREFIX_MAX_ROWS":"32768","TNB_SUFFIX_MAX_ROWS":"32768"}' '{"TNB_PREFIX_MAX_ROWS":"1024","TNB_SUFFIX_MAX_ROWS":"1048576"}' '{"TNB_PREFIX_MAX_ROWS":"1048576","TNB_SUFFIX_MAX_ROWS":"1024"}' '{"TNB_PREFIX_MAX_ROWS":"1024","TNB_SUFFIX_MAX_ROWS":"1024"}' > gpurun_out/sweep_cfg2.txt 2>&1
python tools/bench_entries.py --sweep cfg5 '{}' '{"TNB_PREFIX_MAX_ROWS":"16384"}' '{"TNB_SUFFIX_MAX_ROWS":"128"}' '{"TNB_PREFIX_MAX_ROWS":"16384","TNB_SUFFIX_MAX_ROWS":"128"}' > gpurun_out/sweep_cfg5.txt 2>&1
cat gpurun_out/sweep_cfg2.txt gpurun_out/sweep_cfg5.txt
