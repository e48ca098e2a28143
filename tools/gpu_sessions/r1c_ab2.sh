#!/bin/bash
# Same-box A/B: HEAD build vs new build (lean MMA loop, pre-split halo, 16 KB F16 B stages,
# 8-deep W ring) with grp=1/2 and W ring 4/8.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "edge or index_map or bit_exact or config1 or sharded" > gpurun_out/ab2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab2_pytest.log
for rep in 1 2; do
  ICNNM_LIB_AB=build/ab/libicnnm_b200_head.so timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/ab2_head_$rep.log 2>&1
  ICNNM_TC_GRP=1 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/ab2_g1w8_$rep.log 2>&1
  ICNNM_TC_GRP=1 ICNNM_TC_WS=4 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/ab2_g1w4_$rep.log 2>&1
  ICNNM_TC_GRP=2 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/ab2_g2w8_$rep.log 2>&1
done
