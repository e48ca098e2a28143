#!/bin/bash
# One-graph solve (setup + events + all iterations): stability of the bench steps, full suite.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 120 python tools/profile_step.py --engine f16x3 --iters 3 > gpurun_out/g_first.log 2>&1; echo "rc=$?" >> gpurun_out/g_first.log
for rep in 1 2 3; do timeout 900 python bench.py --no-cpu-baseline > gpurun_out/g_bench_$rep.log 2>&1; done
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/g_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g_pytest.log
