#!/bin/bash
# Tile-group schedule (A chunk shared by two N-tiles, skewed): parity + A/B against grp=1.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python tools/tc_probe.py > gpurun_out/tg_probe.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/tg_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/tg_pytest.log
for v in "1 0" "2 0" "2 2" "2 4"; do set -- $v
  ICNNM_TC_GRP=$1 ICNNM_TC_SKEW=$2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tg_launches_$1_$2.csv python tools/profile_step.py --engine f16x3 --iters 3 > gpurun_out/tg_ncu_$1_$2.log 2>&1
done
for rep in 1 2; do for v in "1 0" "2 4" "2 2"; do set -- $v
  ICNNM_TC_GRP=$1 ICNNM_TC_SKEW=$2 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/tg_bench_$1_$2_$rep.log 2>&1
done; done
