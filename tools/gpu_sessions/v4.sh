#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/v4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/v4_pytest.log
for e in f16x3 tf32x3; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v4_launches_$e.csv python tools/profile_step.py --engine $e --iters 3 > gpurun_out/v4_ncu_$e.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"icnnm_tc_kernel" -s 2 -c 2 -o gpurun_out/prof_${e}_v4 python tools/profile_step.py --engine $e --iters 3 > gpurun_out/v4_ncufull_$e.log 2>&1
done
for rep in 1 2; do
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/v4_bench_f16x3_$rep.log 2>&1
  timeout 900 python bench.py --no-cpu-baseline --engine tf32x3 > gpurun_out/v4_bench_tf32x3_$rep.log 2>&1
done
