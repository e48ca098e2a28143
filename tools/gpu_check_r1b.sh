set -x
python -m pytest tests -m gpu -x -q -k "nccl_one_rank or sharded or exact_residual or config5" > gpurun_out/gpu_tests_new.log 2>&1
tail -3 gpurun_out/gpu_tests_new.log
for v in 1 0 1 0; do ICNNM_GRAPH_SPLIT=$v python bench.py --no-cpu-baseline > gpurun_out/bench_split$v.log 2>&1; tail -1 gpurun_out/bench_split$v.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('split', $v, d['value'], d['e2e']['value'])"; done
ICNNM_TIMING=1 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, time, paper_2604_17001_b200 as P
from paper_2604_17001_b200 import synth
w=synth.WORKLOADS[2]; X=w.target(); m=w.mask(); B=P.learn_ensemble_basis(w.training(), w.kernel)
cfg=P.SolverConfig(max_iters=w.iters, tol_primal=1e-300, tol_change=1e-300)
for i in range(3):
    t=time.perf_counter(); L,r=P.icnnm_solve(X*m,m,B,cfg); print('call',i,(time.perf_counter()-t)*1e3,'ms wall, device',r.device_seconds*1e3)
" > gpurun_out/e2e_timing.log 2>&1
tail -12 gpurun_out/e2e_timing.log
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
