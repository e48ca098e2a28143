#!/bin/bash
# GPU session: CNNM baseline parity + config-2 timing.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_cnnm.py -x -q > gpurun_out/pytest_cnnm.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_cnnm.log
timeout 600 python tools/cnnm_timing.py > gpurun_out/cnnm_timing.log 2>&1
echo "timing rc=$?" >> gpurun_out/cnnm_timing.log
