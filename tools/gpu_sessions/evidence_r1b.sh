#!/bin/bash
# Round-1 evidence: smoke, full GPU suite, default bench (contract line), ncu launch list
# of the bench command, one --set full capture of the two F16x3 contraction kernels.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/e_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e_pytest.log
timeout 900 python bench.py > gpurun_out/e_bench.log 2>&1; echo "rc=$?" >> gpurun_out/e_bench.log
timeout 900 python bench.py --engine tf32x3 --no-cpu-baseline > gpurun_out/e_bench_tf32.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/e_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/e_ncu_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"icnnm_tc_kernel" -s 2 -c 2 -o gpurun_out/prof_f16x3_r1 python tools/profile_step.py --engine f16x3 --iters 3 > gpurun_out/e_ncu_full.log 2>&1
