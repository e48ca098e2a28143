#!/bin/bash
# Final-tree evidence (v10: PDL + graph split + one-rank NCCL transport)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/v10_bench_1.log 2>&1; tail -1 gpurun_out/v10_bench_1.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/v10_bench_2.log 2>&1; tail -1 gpurun_out/v10_bench_2.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/v10_bench_ref.log 2>&1; tail -1 gpurun_out/v10_bench_ref.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/v10_bench_torchrun.log 2>&1; tail -1 gpurun_out/v10_bench_torchrun.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v10_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/v10_ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"icnnm_tc_kernel" -s 2 -c 2 -o gpurun_out/prof_f16x3_v10 python tools/profile_step.py --engine f16x3 --iters 3 > gpurun_out/v10_ncufull.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_extract.py gpurun_out/prof_f16x3_v10.ncu-rep > gpurun_out/v10_ncu_full.json 2>&1; head -c 1500 gpurun_out/v10_ncu_full.json
