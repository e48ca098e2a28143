#!/bin/bash
# e2e host path: upload scan overlapped with the H2D copies, basis-validation cache
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v10f_gpu_tests.log 2>&1; tail -n 3 gpurun_out/v10f_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v10f_smoke.log 2>&1; tail -n 1 gpurun_out/v10f_smoke.log
timeout 900 python bench.py > gpurun_out/v10f_bench.log 2>&1; tail -n 1 gpurun_out/v10f_bench.log
ICNNM_TIMING=1 timeout 300 python tools/e2e_breakdown.py > gpurun_out/v10f_e2e_breakdown.log 2>&1; tail -n 24 gpurun_out/v10f_e2e_breakdown.log
