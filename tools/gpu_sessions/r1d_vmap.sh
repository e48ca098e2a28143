#!/bin/bash
# Voxel order within a brick (vmap 1: warps' two 16-t runs one h-row apart -> conflict-free
# halo gathers / col2im scatter at config 2): exactness, parity subset, same-box A/B, ncu conflicts.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "edge or index_map or bit_exact or config1 or golden or cluster or sharded or adjointness" > gpurun_out/u_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/u_pytest.log
for rep in 1 2 3; do
  ICNNM_TC_VMAP=0 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/u_v0_$rep.log 2>&1
  timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/u_v1_$rep.log 2>&1
done
for v in 0 1; do
  ICNNM_TC_VMAP=$v timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none -k regex:"icnnm_tc_kernel" -s 2 -c 2 --csv --log-file gpurun_out/u_ncu_v$v.csv python tools/profile_step.py --engine f16x3 --iters 3 > gpurun_out/u_ncu_v$v.log 2>&1
done
