timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -5
python bench.py --no-cpu-baseline > gpurun_out/s4_bench4.json 2> gpurun_out/s4_bench4.err
python bench.py --config 2 --no-cpu-baseline > gpurun_out/s4_bench2.json 2> gpurun_out/s4_bench2.err
python tools/with_ab_lib.py tools/tc_counters.py --config 4 --iters 20 2>&1 | head -3
