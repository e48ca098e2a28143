#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python tools/measure_peaks.py > gpurun_out/peaks.json 2> gpurun_out/peaks.err
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_r4.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r4.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_r4.log
timeout 300 python tools/profile_step.py --engine tf32x3 --iters 3 > gpurun_out/plain_tc.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tc_r4.csv python tools/profile_step.py --engine tf32x3 --iters 3 > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"icnnm_tc_kernel" -s 2 -c 2 -o gpurun_out/prof_tc_r4 python tools/profile_step.py --engine tf32x3 --iters 3 > gpurun_out/ncu_full.log 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
