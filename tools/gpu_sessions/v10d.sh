#!/bin/bash
# forward tile groups (ICNNM_TC_GRP=2: both N-tiles share every built A chunk) at configs 4 and 3
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/ab_grp
for v in 2 -1 2 -1; do
  if [ "$v" = "-1" ]; then unset ICNNM_TC_GRP; else export ICNNM_TC_GRP=$v; fi
  timeout 900 python bench.py --config 4 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/ab_grp/cfg4_grp$v.log 2>&1
  tail -n 1 gpurun_out/ab_grp/cfg4_grp$v.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg4 grp', '$v', d['value'], d['roofline']['per_launch_ms'], d['clocks']['sm_mhz'])"
done
unset ICNNM_TC_GRP
for v in 2 -1; do
  if [ "$v" = "-1" ]; then unset ICNNM_TC_GRP; else export ICNNM_TC_GRP=$v; fi
  timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/ab_grp/cfg3_grp$v.log 2>&1
  tail -n 1 gpurun_out/ab_grp/cfg3_grp$v.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg3 grp', '$v', d['value'], d['roofline']['per_launch_ms'], d['clocks']['sm_mhz'])"
done
