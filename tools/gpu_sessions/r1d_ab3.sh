#!/bin/bash
# Same-box A/B: incremental builder stage counters vs HEAD; parity subset.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "edge or index_map or bit_exact or config1 or golden" > gpurun_out/v_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/v_pytest.log
for rep in 1 2 3; do
  ICNNM_LIB_AB=build/ab/libicnnm_b200_head.so timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/v_head_$rep.log 2>&1
  timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/v_new_$rep.log 2>&1
done
