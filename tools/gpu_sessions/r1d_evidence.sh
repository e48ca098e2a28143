#!/bin/bash
# Re-entry evidence on HEAD: GPU suite, smoke, bench x2, bench launch list, --set full of the TC kernels.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/d_smi.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/d_smoke.log
for rep in 1 2; do timeout 900 python bench.py > gpurun_out/d_bench_$rep.log 2>&1; echo "rc=$?" >> gpurun_out/d_bench_$rep.log; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/d_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/d_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"icnnm_tc_kernel" -s 2 -c 2 -o gpurun_out/prof_f16x3_d python tools/profile_step.py --engine f16x3 --iters 3 > gpurun_out/d_ncu_full.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/d_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/d_pytest.log
