#!/bin/bash
# A/B: 2x2x32 bricks (conflict-free gathers/scatter) vs 2x4x16.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python tools/tc_probe.py > gpurun_out/bt_probe.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/bt_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/bt_pytest.log
for v in 1 0; do for e in f16x3 tf32x3; do
  ICNNM_TC_BT32=$v timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none --csv --log-file gpurun_out/bt_launches_${e}_$v.csv python tools/profile_step.py --engine $e --iters 3 > gpurun_out/bt_ncu_${e}_$v.log 2>&1
done; done
for rep in 1 2; do for v in 1 0; do
  ICNNM_TC_BT32=$v timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bt_bench_${v}_$rep.log 2>&1
done; done
