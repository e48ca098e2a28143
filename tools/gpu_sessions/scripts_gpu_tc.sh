#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 120 python tools/tc_probe.py > gpurun_out/tc_probe.log 2>&1; echo "rc=$?" >> gpurun_out/tc_probe.log
