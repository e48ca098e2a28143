timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "gram or learn_basis" 2>&1 | tail -3
timeout 120 python tools/gram_profile.py --config 2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:gram --log-file gpurun_out/s10_gram_launches2.csv python tools/gram_profile.py --config 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:gram --log-file gpurun_out/s10_gram_launches3.csv python tools/gram_profile.py --config 3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:gram --log-file gpurun_out/s10_gram_launches5.csv python tools/gram_profile.py --config 5 > /dev/null 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s10_bench4.json 2> gpurun_out/s10_bench4.err
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/s10_bench2.json 2> gpurun_out/s10_bench2.err
