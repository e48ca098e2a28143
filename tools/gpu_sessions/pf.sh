#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for e in f16x3 tf32x3; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pf_launches_$e.csv python tools/profile_step.py --engine $e --iters 3 > gpurun_out/pf_ncu_$e.log 2>&1
  ICNNM_TC_SKIP=64 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pf_launches_${e}_off.csv python tools/profile_step.py --engine $e --iters 3 > gpurun_out/pf_ncu_${e}_off.log 2>&1
  ICNNM_TC_SB=4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pf_launches_${e}_sb4.csv python tools/profile_step.py --engine $e --iters 3 > gpurun_out/pf_ncu_${e}_sb4.log 2>&1
  ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine $e --iters 5 --runs 2 > gpurun_out/pf_counters_$e.log 2>&1
done
