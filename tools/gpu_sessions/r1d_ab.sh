#!/bin/bash
# e2e phase breakdown; CTA pairs vs single CTAs (same box); B-stream cost (SKIP=4: no B copies).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python tools/e2e_breakdown.py > gpurun_out/e_breakdown.log 2>&1
for rep in 1 2; do
  for v in "1 0 0" "2 0 0" "2 12 0" "1 0 4"; do set -- $v
    env ICNNM_TC_CS=$1 $( [ $2 -gt 0 ] && echo ICNNM_TC_SB=$2 ) ICNNM_TC_SKIP=$3 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/e_ab_$1_$2_$3_$rep.log 2>&1
  done
done
for cs in 1 2; do
  ICNNM_TC_CS=$cs ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine f16x3 --iters 5 --runs 2 > gpurun_out/e_counters_$cs.log 2>&1
done
