#!/bin/bash
# A/B of the forward/adjoint A-operand build modes (alternate-chunk groups vs split chunks).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python tools/tc_probe.py > gpurun_out/ab_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tc or tf32 or engine or solve_cfg1" > gpurun_out/ab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab_pytest.log
for mode in 0 1; do
  ICNNM_TC_BSPLIT=$mode ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine tf32x3 --iters 5 --runs 2 > gpurun_out/ab_counters_$mode.log 2>&1
  ICNNM_TC_BSPLIT=$mode timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_launches_$mode.csv python tools/profile_step.py --engine tf32x3 --iters 3 > gpurun_out/ab_ncu_$mode.log 2>&1
done
for rep in 1 2; do for mode in 0 1; do
  ICNNM_TC_BSPLIT=$mode timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_bench_${mode}_$rep.log 2>&1
done; done
