#!/bin/bash
# Knob A/B on the new epilogues: forward tile groups (A reuse), skew, B ring depth; update-kernel ncu.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for rep in 1 2; do
  timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/t_base_$rep.log 2>&1
  ICNNM_TC_GRP=2 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/t_grp2_$rep.log 2>&1
  ICNNM_TC_GRP=2 ICNNM_TC_SKEW=2 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/t_grp2s2_$rep.log 2>&1
  ICNNM_TC_SB=6 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/t_sb6_$rep.log 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:"icnnm_update|icnnm_coef" -s 4 -c 2 -o gpurun_out/prof_update python tools/profile_step.py --engine f16x3 --iters 3 > gpurun_out/t_ncu_update.log 2>&1
