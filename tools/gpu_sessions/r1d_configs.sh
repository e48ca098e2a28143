#!/bin/bash
# BASELINE configs 1, 3 and 4 at N=1 (informative; the headline is config 2).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c_cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/c_cfg3.log
timeout 1200 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c_cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/c_cfg4.log
timeout 600 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c_cfg1.log 2>&1; echo "rc=$?" >> gpurun_out/c_cfg1.log
