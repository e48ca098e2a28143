#!/bin/bash
# update kernel (one wave, 4 elements in flight), 6-stage B default, SB=8 A/B;
# CTA pairs with CTA-scope waits (skip bit 64): correctness probe + timing.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
ICNNM_TC_CS=2 ICNNM_TC_SKIP=64 timeout 120 python tools/f16_pair_probe.py > gpurun_out/w_probe.log 2>&1; echo "rc=$?" >> gpurun_out/w_probe.log
for rep in 1 2; do
  timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/w_base_$rep.log 2>&1
  ICNNM_TC_SB=8 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/w_sb8_$rep.log 2>&1
  ICNNM_TC_CS=2 ICNNM_TC_SKIP=64 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/w_pair64_$rep.log 2>&1
done
ICNNM_TC_CS=2 ICNNM_TC_SKIP=64 ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine f16x3 --iters 5 --runs 2 > gpurun_out/w_counters_pair64.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"icnnm_update" -s 2 -c 1 -o gpurun_out/prof_update2 python tools/profile_step.py --engine f16x3 --iters 3 > gpurun_out/w_ncu_update.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "edge or index_map or bit_exact or config1 or sharded or golden" > gpurun_out/w_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/w_pytest.log
