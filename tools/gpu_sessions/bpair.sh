#!/bin/bash
# A/B: builder chunk pairing (one wait::st per two owned chunks) + vectorised tap loads.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python tools/tc_probe.py > gpurun_out/bp_probe.log 2>&1
ICNNM_TC_BPAIR=1 timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/bp_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/bp_pytest.log
for v in 1 0; do for e in f16x3 tf32x3; do
  ICNNM_TC_BPAIR=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bp_launches_${e}_$v.csv python tools/profile_step.py --engine $e --iters 3 > gpurun_out/bp_ncu_${e}_$v.log 2>&1
  ICNNM_TC_BPAIR=$v ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine $e --iters 5 --runs 2 > gpurun_out/bp_counters_${e}_$v.log 2>&1
done; done
for rep in 1 2; do for v in 1 0; do
  ICNNM_TC_BPAIR=$v timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bp_bench_${v}_$rep.log 2>&1
done; done
