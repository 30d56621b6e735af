cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 600 python tools/entries_wall_probe.py > gpurun_out/wall_probe.txt 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo "rc=$?" >> gpurun_out/bench_r02a.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_r02a.json 2>&1
python tools/write_peak.py > gpurun_out/write_peak.txt 2>&1
cat gpurun_out/wall_probe.txt gpurun_out/write_peak.txt; tail -3 gpurun_out/bench_r02a.err; cut -c1-3000 gpurun_out/bench_r02a.json; cut -c1-600 gpurun_out/ref_r02a.json
