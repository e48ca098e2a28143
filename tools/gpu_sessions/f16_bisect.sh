#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python tools/f16_bisect.py > gpurun_out/f16_bisect.log 2>&1
