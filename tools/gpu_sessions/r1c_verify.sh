#!/bin/bash
# Re-entry verification of HEAD: smoke, full GPU suite, default bench, BPAIR A/B bench.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/v_smi.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/v_bench.log 2>&1; echo "rc=$?" >> gpurun_out/v_bench.log
ICNNM_TC_BPAIR=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/v_bench_bpair.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/v_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/v_pytest.log
