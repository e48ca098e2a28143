#!/bin/bash
# cta_group::2 CTA pairs: first contact with short timeouts, then parity and A/B.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
ICNNM_TC_CS=1 timeout 120 python tools/profile_step.py --engine f16x3 --iters 3 > gpurun_out/p_cs1.log 2>&1; echo "rc=$?" >> gpurun_out/p_cs1.log
timeout 90 python tools/f16_pair_probe.py > gpurun_out/p_probe.log 2>&1; echo "rc=$?" >> gpurun_out/p_probe.log
if grep -q "rc=0" gpurun_out/p_probe.log; then
  timeout 120 python tools/profile_step.py --engine f16x3 --iters 3 > gpurun_out/p_cs2.log 2>&1; echo "rc=$?" >> gpurun_out/p_cs2.log
  timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "edge or index_map or bit_exact or config1 or sharded or golden or small" > gpurun_out/p_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p_pytest.log
  for rep in 1 2; do
    ICNNM_TC_CS=1 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/p_b1_$rep.log 2>&1
    timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/p_b2_$rep.log 2>&1
  done
fi
