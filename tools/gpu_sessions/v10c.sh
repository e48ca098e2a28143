#!/bin/bash
# config-5 recipe on one GPU through the NCCL transport; informative config 1/3/4 lines
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python bench.py --config 5 --dims 128 1024 64 --steps 3 --warmup 3 > gpurun_out/v10c_cfg5_128.log 2>&1; tail -n 1 gpurun_out/v10c_cfg5_128.log
timeout 900 python bench.py --config 5 --dims 256 1024 64 --steps 3 --warmup 3 > gpurun_out/v10c_cfg5_256.log 2>&1; tail -n 1 gpurun_out/v10c_cfg5_256.log
for c in 1 3 4; do timeout 1200 python bench.py --config $c --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/v10c_cfg$c.log 2>&1; tail -n 1 gpurun_out/v10c_cfg$c.log | cut -c1-300; done
