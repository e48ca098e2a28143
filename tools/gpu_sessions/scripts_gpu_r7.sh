#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_r7.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_r7.log
timeout 300 python tools/profile_step.py --engine tf32x3 --iters 3 > gpurun_out/plain_tc.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"icnnm_tc_kernel" -s 2 -c 2 -o gpurun_out/prof_tc_r7 python tools/profile_step.py --engine tf32x3 --iters 3 > gpurun_out/ncu_full.log 2>&1
