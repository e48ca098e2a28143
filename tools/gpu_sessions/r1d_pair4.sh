#!/bin/bash
# CTA pairs: B ring depth (half stages), same box vs single.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for rep in 1 2; do
  timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/r_base_$rep.log 2>&1
  ICNNM_TC_CS=2 ICNNM_TC_SB=12 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/r_pair12_$rep.log 2>&1
  ICNNM_TC_CS=2 ICNNM_TC_SB=10 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/r_pair10_$rep.log 2>&1
  ICNNM_TC_CS=2 ICNNM_TC_SB=12 ICNNM_TC_GRP=2 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/r_pair12g2_$rep.log 2>&1
done
ICNNM_TC_CS=2 ICNNM_TC_SB=12 ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine f16x3 --iters 5 --runs 2 > gpurun_out/r_counters_pair12.log 2>&1
