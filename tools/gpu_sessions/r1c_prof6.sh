#!/bin/bash
# v6 evidence: in-kernel role counters, launch list, one --set full capture (source-level)
# of the forward and adjoint F16x3 kernels, then the full GPU suite.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine f16x3 --iters 5 --runs 2 > gpurun_out/p6_counters.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p6_launches.csv python tools/profile_step.py --engine f16x3 --iters 3 > gpurun_out/p6_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"icnnm_tc_kernel" -s 2 -c 2 -o gpurun_out/prof_f16x3_v6 python tools/profile_step.py --engine f16x3 --iters 3 > gpurun_out/p6_ncu_full.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/p6_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p6_pytest.log
