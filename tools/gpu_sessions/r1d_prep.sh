#!/bin/bash
# Builder time split (chunk waits / chunk work / per-brick prep / other) for both kernels.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine f16x3 --iters 5 --runs 2 > gpurun_out/p_counters.log 2>&1
ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --config 4 --engine f16x3 --iters 5 --runs 2 > gpurun_out/p_counters_cfg4.log 2>&1
