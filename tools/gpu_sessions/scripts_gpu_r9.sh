#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "config1 or handle or exact or objective_trace or cosine" --timeout 300 > gpurun_out/pytest_sub.log 2>&1
for i in 1 2 3; do timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r9_$i.log 2>&1; done
