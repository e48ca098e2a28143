#!/bin/bash
# device cache + lazy packing: e2e breakdown, bench (with e2e), pair builder isolation, GPU suite.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python tools/e2e_breakdown.py > gpurun_out/f_breakdown.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/f_bench.log 2>&1
for cs in 1 2; do
  ICNNM_TC_CS=$cs ICNNM_TC_SKIP=1 ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine f16x3 --iters 5 --runs 2 > gpurun_out/f_counters_skip1_$cs.log 2>&1
done
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f_pytest.log
