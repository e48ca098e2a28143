#!/bin/bash
# Source-level ncu capture of the CTA-pair kernels (where does the pipeline stall?).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
ICNNM_TC_CS=2 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"icnnm_tc_kernel" -s 2 -c 2 -o gpurun_out/prof_pair python tools/profile_step.py --engine f16x3 --iters 3 > gpurun_out/pp_ncu.log 2>&1
