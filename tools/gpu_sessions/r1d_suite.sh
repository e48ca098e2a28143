#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/y_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/y_smoke.log
timeout 300 python tools/e2e_breakdown.py > gpurun_out/y_breakdown.log 2>&1
timeout 900 python bench.py > gpurun_out/y_bench.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/y_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/y_pytest.log
