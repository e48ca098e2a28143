#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 120 python tools/tc_probe.py > gpurun_out/tc_probe.log 2>&1
ICNNM_TC_COUNTERS=1 timeout 120 python tools/profile_step.py --engine tf32x3 --iters 5 --runs 2 > gpurun_out/tc_skip.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "adjoint or recipe or config1 or sharded" --timeout 300 > gpurun_out/pytest_sub.log 2>&1
