#!/bin/bash
# Tight B stage stride (13 KB at wbase 208): deeper rings fit.  Same-box A/B vs HEAD.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "edge or index_map or bit_exact or config1 or golden or cluster" > gpurun_out/b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/b_pytest.log
for rep in 1 2; do
  ICNNM_LIB_AB=build/ab/libicnnm_b200_head.so timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/b_head_$rep.log 2>&1
  timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/b_new_$rep.log 2>&1
  ICNNM_TC_SB=10 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/b_sb10_$rep.log 2>&1
  ICNNM_TC_SB=12 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/b_sb12_$rep.log 2>&1
done
