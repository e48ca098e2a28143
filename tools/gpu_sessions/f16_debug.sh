#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python tools/f16_debug.py > gpurun_out/f16_debug.log 2>&1
for e in f16x3 tf32x3; do
  ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine $e --iters 5 --runs 2 > gpurun_out/f16b_counters_$e.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f16b_launches_$e.csv python tools/profile_step.py --engine $e --iters 3 > gpurun_out/f16b_ncu_$e.log 2>&1
done
