#!/bin/bash
# End-of-session evidence on the final tree: smoke, GPU suite, bench x2, reference arm,
# bench launch list, --set full of the TC kernels, update-kernel capture.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/zz_smi.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/zz_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/zz_smoke.log
for rep in 1 2; do timeout 900 python bench.py > gpurun_out/zz_bench_$rep.log 2>&1; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/zz_ref.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 2 --warmup 3 > gpurun_out/zz_torchrun.log 2>&1; echo "rc=$?" >> gpurun_out/zz_torchrun.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29518 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/zz_torchrun_ref.log 2>&1; echo "rc=$?" >> gpurun_out/zz_torchrun_ref.log
timeout 300 python tools/e2e_breakdown.py > gpurun_out/zz_breakdown.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/zz_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/zz_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"icnnm_tc_kernel|icnnm_update" -s 3 -c 3 -o gpurun_out/prof_final2 python tools/profile_step.py --engine f16x3 --iters 3 > gpurun_out/zz_ncu_full.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/zz_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/zz_pytest.log
