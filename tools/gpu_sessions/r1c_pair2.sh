#!/bin/bash
# CTA pairs: role counters and B-ring depth (half-size stages), vs single CTAs.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 90 python tools/f16_pair_probe.py > gpurun_out/q_probe.log 2>&1; echo "rc=$?" >> gpurun_out/q_probe.log
for v in "2 8" "2 12" "1 4"; do set -- $v
  ICNNM_TC_CS=$1 ICNNM_TC_SB=$2 ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine f16x3 --iters 5 --runs 2 > gpurun_out/q_counters_$1_$2.log 2>&1
  ICNNM_TC_CS=$1 ICNNM_TC_SB=$2 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/q_b_$1_$2.log 2>&1
done
