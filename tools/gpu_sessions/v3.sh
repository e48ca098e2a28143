#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python tools/tc_probe.py > gpurun_out/v3_probe.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/v3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/v3_pytest.log
for e in f16x3 tf32x3; do
  ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine $e --iters 5 --runs 2 > gpurun_out/v3_counters_$e.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v3_launches_$e.csv python tools/profile_step.py --engine $e --iters 3 > gpurun_out/v3_ncu_$e.log 2>&1
done
for rep in 1 2; do for e in f16x3 tf32x3; do
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --engine $e > gpurun_out/v3_bench_${e}_$rep.log 2>&1
done; done
