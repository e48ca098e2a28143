#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
(timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e ; echo "rc=$?") > gpurun_out/b_cfg2.log 2>&1
(timeout 600 python bench.py --config 4 --iters 20 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ; echo "rc=$?") > gpurun_out/b_cfg4.log 2>&1
(timeout 600 python bench.py --config 5 --dims 128 128 64 --iters 20 --steps 1 --warmup 3 ; echo "rc=$?") > gpurun_out/b_cfg5.log 2>&1
(timeout 900 python bench.py --config 3 --iters 20 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ; echo "rc=$?") > gpurun_out/b_cfg3.log 2>&1
(timeout 300 python bench.py --config 5 --steps 1 --warmup 3 ; echo "rc=$?") > gpurun_out/b_cfg5full.log 2>&1
