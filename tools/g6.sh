cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 300 python tools/widen_probe.py > gpurun_out/widen_probe2.txt 2>&1
for f in 0 0.3; do TNB_E2E_TRACE=1 TNB_E2E_RAW_FRAC=$f timeout 300 python -c "
import os,sys,time,torch
sys.path.insert(0,'.')
import paper_2206_11128_b200 as tb, workloads as W
from paper_2206_11128_b200 import core as C
m=1<<24; shape=W.CONFIGS['cfg2'][1]
t=tb.TnTensor([tb.ModeNode('tt',c) for c in W.tt_cores(shape,32,0)])
ih=torch.from_numpy(W.indices(shape,m,2)).pin_memory(); po=torch.empty(m).pin_memory()
for i in range(4):
    torch.cuda.synchronize(); t0=time.perf_counter(); tb.entries(t,ih,out=po); torch.cuda.synchronize(); print('raw_frac $f e2e ms', (time.perf_counter()-t0)*1e3, C.last_transfer, flush=True)
" >> gpurun_out/e2e_trace.txt 2>&1; done
P="python bench.py --op full --steps 2 --warmup 1 --no-cpu"
for v in 0 1; do
  TNB_FULL_TMA_STORE=$v timeout 300 $P > gpurun_out/pf$v.log 2>&1 && \
  TNB_FULL_TMA_STORE=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:full_tc -s 1 -c 1 \
    -o gpurun_out/prof_full_tma$v $P > gpurun_out/ncu_full_tma$v.log 2>&1
  echo "ncu $v rc=$?" >> gpurun_out/ncu_full_tma$v.log
done
cat gpurun_out/widen_probe2.txt gpurun_out/e2e_trace.txt; tail -2 gpurun_out/ncu_full_tma*.log; ls -la gpurun_out/*.ncu-rep
