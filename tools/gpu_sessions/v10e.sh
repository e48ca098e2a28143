#!/bin/bash
# compute-sanitizer on the final tree (PDL edges on): memcheck + synccheck, small solves
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/v10e_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -n 6 gpurun_out/v10e_memcheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/v10e_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -n 6 gpurun_out/v10e_synccheck.log
