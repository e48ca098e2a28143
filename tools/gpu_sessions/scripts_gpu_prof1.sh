#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python tools/measure_peaks.py > gpurun_out/peaks.json 2> gpurun_out/peaks.err
for E in tf32x3 ffma; do
  timeout 300 python tools/profile_step.py --engine $E --iters 3 > gpurun_out/plain_$E.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$E.csv python tools/profile_step.py --engine $E --iters 3 > gpurun_out/ncu_list_$E.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"icnnm_tc_kernel|icnnm_fwd_ffma|icnnm_adj_ffma" -s 2 -c 2 -o gpurun_out/prof_$E python tools/profile_step.py --engine $E --iters 3 > gpurun_out/ncu_full_$E.log 2>&1
done
