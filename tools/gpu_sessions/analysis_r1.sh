#!/bin/bash
# GPU session: analyze-path parity + timing on config 2.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_analysis.py -x -q > gpurun_out/pytest_analysis.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_analysis.log
timeout 300 python tools/analyze_timing.py --config 2 > gpurun_out/analyze_timing.log 2>&1
echo "timing rc=$?" >> gpurun_out/analyze_timing.log
