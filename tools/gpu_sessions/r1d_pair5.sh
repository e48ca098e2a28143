#!/bin/bash
# CTA pairs with relay-free B halves (2-SM tensor copies into the leader's barrier).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
ICNNM_TC_CS=2 timeout 180 python tools/f16_pair_probe.py > gpurun_out/x_probe.log 2>&1; echo "rc=$?" >> gpurun_out/x_probe.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster" > gpurun_out/x_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/x_pytest.log
for rep in 1 2; do
  timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/x_base_$rep.log 2>&1
  ICNNM_TC_CS=2 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/x_tma8_$rep.log 2>&1
  ICNNM_TC_CS=2 ICNNM_TC_SB=12 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/x_tma12_$rep.log 2>&1
  ICNNM_TC_CS=2 ICNNM_TC_SB=12 ICNNM_TC_TMAPAIR=0 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/x_relay12_$rep.log 2>&1
done
ICNNM_TC_CS=2 ICNNM_TC_SB=12 ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine f16x3 --iters 5 --runs 2 > gpurun_out/x_counters.log 2>&1
