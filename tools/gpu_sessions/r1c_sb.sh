#!/bin/bash
# B-ring depth A/B (pairs on/off), same box.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for rep in 1 2; do
  for v in "4 8 2" "6 8 2" "6 6 2" "8 4 2" "6 8 1"; do set -- $v
    ICNNM_TC_SB=$1 ICNNM_TC_WS=$2 ICNNM_TC_CS=$3 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/sb_$1_$2_$3_$rep.log 2>&1
  done
done
ICNNM_TC_SB=6 ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine f16x3 --iters 5 --runs 2 > gpurun_out/sb_counters.log 2>&1
