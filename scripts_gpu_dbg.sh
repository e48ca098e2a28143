#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 120 python tools/tc_probe.py > gpurun_out/tc_probe.log 2>&1
for S in 0; do echo "skip=$S" ; ICNNM_TC_SKIP=$S ICNNM_TC_COUNTERS=1 timeout 120 python tools/profile_step.py --engine tf32x3 --iters 5 --runs 2 ; done > gpurun_out/tc_skip.log 2>&1
