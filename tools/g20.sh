cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export TNB_BENCH_BACKEND=gloo
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-secondary > gpurun_out/bench_n2_entries.json 2> gpurun_out/bench_n2_entries.err; echo "rc=$?" >> gpurun_out/bench_n2_entries.err
timeout 600 python bench.py --gpus 2 --op full --steps 3 --warmup 3 > gpurun_out/bench_n2_full.json 2> gpurun_out/bench_n2_full.err; echo "rc=$?" >> gpurun_out/bench_n2_full.err
timeout 600 python bench.py --gpus 2 --op dot --steps 3 --warmup 3 > gpurun_out/bench_n2_dot.json 2> gpurun_out/bench_n2_dot.err; echo "rc=$?" >> gpurun_out/bench_n2_dot.err
timeout 600 python bench.py --gpus 2 --impl reference --steps 2 --warmup 1 > gpurun_out/bench_n2_ref.json 2> gpurun_out/bench_n2_ref.err; echo "rc=$?" >> gpurun_out/bench_n2_ref.err
for f in entries full dot ref; do echo "== $f"; tail -2 gpurun_out/bench_n2_$f.err; cut -c1-700 gpurun_out/bench_n2_$f.json; done
