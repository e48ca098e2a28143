#!/bin/bash
# Cost breakdown by removing work (timing experiments only): skip 1 = no A build work,
# 2 = no epilogue work, 4 = no B copies; plus the new stage selection (SB 4/6).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for v in 0 4 1 2 6 7; do
  ICNNM_TC_SKIP=$v timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/skip_$v.log 2>&1
done
for sb in 4 6 8; do
  ICNNM_TC_SB=$sb timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/sbn_$sb.log 2>&1
done
