# per-role phase times of the global-sort compute kernel (cfg2, cfg5 with TNB_ENTRIES_GSORT=2)
[ -f build/variants/trace/libtnb.so ] || python tools/build_variant.py trace -DTNB_GS_TRACE=1
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
TNB_LIB=build/variants/trace/libtnb.so TNB_GS_TRACE_FILE=gpurun_out/gs_cfg2.trace python tools/bench_entries.py --one cfg2 | cut -c1-200
python tools/gs_trace.py gpurun_out/gs_cfg2.trace 885.6
TNB_ENTRIES_GSORT=2 TNB_LIB=build/variants/trace/libtnb.so TNB_GS_TRACE_FILE=gpurun_out/gs_cfg5.trace python tools/bench_entries.py --one cfg5 | cut -c1-200
python tools/gs_trace.py gpurun_out/gs_cfg5.trace 3542.5
