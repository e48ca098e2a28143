#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
ICNNM_TC_PAIR=1 timeout 90 python tools/tc_probe.py > gpurun_out/tc_probe_pair.log 2>&1; echo "rc=$?" >> gpurun_out/tc_probe_pair.log
if grep -q "rc=0" gpurun_out/tc_probe_pair.log; then
  for P in 0 1; do echo "pair=$P"; ICNNM_TC_PAIR=$P ICNNM_TC_COUNTERS=1 timeout 120 python tools/profile_step.py --engine tf32x3 --iters 5 --runs 2; done > gpurun_out/tc_pair_cmp.log 2>&1
fi
