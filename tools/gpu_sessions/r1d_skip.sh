#!/bin/bash
# Where do the cycles go (timing only, results invalid under SKIP): 1 = no A build,
# 2 = no epilogue work, 4 = no B copies, combos.  Plus the cluster-mode subprocess tests.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster_modes" > gpurun_out/s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s_pytest.log
for sk in 0 1 2 4 3 6 7; do
  ICNNM_TC_SKIP=$sk timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s_skip_$sk.log 2>&1
done
