#!/bin/bash
# CTA pairs / B multicast with CTA-scope remote arrives and waits (no MEMBAR.ALL.GPU, no CCTL.IVALL).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster" > gpurun_out/q_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q_pytest.log
for rep in 1 2; do
  timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/q_base_$rep.log 2>&1
  ICNNM_TC_CS=2 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/q_pair_$rep.log 2>&1
  ICNNM_TC_MCB=1 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/q_mcb_$rep.log 2>&1
done
ICNNM_TC_CS=2 ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine f16x3 --iters 5 --runs 2 > gpurun_out/q_counters_pair.log 2>&1
