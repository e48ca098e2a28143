#!/bin/bash
# B multicast across 2-CTA clusters (ICNNM_TC_MCB=1): probe, parity subset, same-box A/B, counters.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
ICNNM_TC_MCB=1 timeout 120 python tools/f16_pair_probe.py > gpurun_out/m_probe.log 2>&1; echo "rc=$?" >> gpurun_out/m_probe.log
ICNNM_TC_MCB=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "edge or index_map or bit_exact or config1 or golden" > gpurun_out/m_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/m_pytest.log
for rep in 1 2; do
  timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/m_base_$rep.log 2>&1
  ICNNM_TC_MCB=1 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/m_mcb_$rep.log 2>&1
done
ICNNM_TC_MCB=1 ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine f16x3 --iters 5 --runs 2 > gpurun_out/m_counters_mcb.log 2>&1
