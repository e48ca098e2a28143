#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for i in 1 2 3; do timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_r12_$i.log 2>&1; done
timeout 300 python tools/profile_step.py --engine tf32x3 --iters 3 > gpurun_out/plain_tc.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tc_r12.csv python tools/profile_step.py --engine tf32x3 --iters 3 > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"icnnm_tc_kernel" -s 2 -c 2 -o gpurun_out/prof_tc_r12 python tools/profile_step.py --engine tf32x3 --iters 3 > gpurun_out/ncu_full.log 2>&1
