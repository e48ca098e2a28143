# PDL A/B on the current tree: parity subset with PDL on, then bench alternating
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_c.log 2>&1; tail -1 gpurun_out/smoke_c.log
python -m pytest tests -m gpu -x -q -k "solve or parity or recipe or exact or nccl or sharded or cnnm" > gpurun_out/gpu_tests_c.log 2>&1
tail -3 gpurun_out/gpu_tests_c.log
for v in 1 0 1 0; do ICNNM_PDL=$v python bench.py --no-cpu-baseline > gpurun_out/bench_pdl$v.log 2>&1; tail -1 gpurun_out/bench_pdl$v.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('pdl', $v, d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], d['roofline']['per_launch_ms'])"; done
for v in 1 0; do ICNNM_PDL=$v python bench.py --config 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c1_pdl$v.log 2>&1; tail -1 gpurun_out/bench_c1_pdl$v.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg1 pdl', $v, d['value'])"; done
