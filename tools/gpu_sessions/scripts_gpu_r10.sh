#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k "edge" --timeout 300 > gpurun_out/pytest_edge.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_edge.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_torchrun.log 2>&1; echo "rc=$?" >> gpurun_out/bench_torchrun.log
