#!/bin/bash
# CTA-pair multicast B stream: first contact (short timeouts), parity subset, same-box A/B.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 120 python tools/profile_step.py --engine f16x3 --iters 3 > gpurun_out/cs_first.log 2>&1; echo "rc=$?" >> gpurun_out/cs_first.log
if grep -q "rc=0" gpurun_out/cs_first.log; then
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "edge or index_map or bit_exact or config1 or sharded or golden or small" > gpurun_out/cs_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/cs_pytest.log
for rep in 1 2; do
  ICNNM_TC_CS=1 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/cs_1_$rep.log 2>&1
  timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/cs_2_$rep.log 2>&1
done
ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine f16x3 --iters 5 --runs 2 > gpurun_out/cs_counters.log 2>&1
fi
