#!/bin/bash
# Final tree: full GPU suite + smoke; config-5 recipe on one GPU through the NCCL transport
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v10b_gpu_tests.log 2>&1; tail -n 3 gpurun_out/v10b_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v10b_smoke.log 2>&1; tail -n 1 gpurun_out/v10b_smoke.log
timeout 900 python bench.py --config 5 --dims 128 1024 64 --steps 3 --warmup 3 > gpurun_out/v10b_cfg5_128.log 2>&1; tail -n 1 gpurun_out/v10b_cfg5_128.log
timeout 900 python bench.py --config 5 --dims 256 1024 64 --steps 3 --warmup 3 > gpurun_out/v10b_cfg5_256.log 2>&1; tail -n 1 gpurun_out/v10b_cfg5_256.log
