timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -5
for c in 4 2 3; do timeout 300 python tools/with_ab_lib.py tools/tc_counters.py --config $c --iters 10 2>&1 | head -1 | sed -e 's/np.float64(//g; s/)//g'; done
timeout 120 python tools/gram_profile.py --config 2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:gram --log-file gpurun_out/s9_gram_launches2.csv python tools/gram_profile.py --config 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:gram --log-file gpurun_out/s9_gram_launches3.csv python tools/gram_profile.py --config 3 > /dev/null 2>&1
