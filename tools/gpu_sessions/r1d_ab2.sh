#!/bin/bash
# Same-box A/B: HEAD kernels vs 8-warp adjoint epilogue (EHALF=2/1) + atomic-free forward norms.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "edge or index_map or bit_exact or config1 or sharded or golden" > gpurun_out/g_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g_pytest.log
for rep in 1 2; do
  ICNNM_LIB_AB=build/ab/libicnnm_b200_head.so timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/g_head_$rep.log 2>&1
  timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/g_new_$rep.log 2>&1
  ICNNM_TC_EHALF=1 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/g_eh1_$rep.log 2>&1
done
ICNNM_TC_COUNTERS=1 timeout 300 python tools/profile_step.py --engine f16x3 --iters 5 --runs 2 > gpurun_out/g_counters.log 2>&1
