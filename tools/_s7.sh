timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "gram or learn_basis or default_config or f64_engine or auto_engine or exact_residual or solve_errors" 2>&1 | tail -15
run() { echo "=== $*"; timeout 120 env "$@" python tools/with_ab_lib.py tools/tc_counters.py --config 4 --iters 20 2>&1 | head -3 | sed -e 's/np.float64(//g; s/)//g'; }
run A=0
run ICNNM_TC_SKIP=56
run ICNNM_TC_SKIP=48
run ICNNM_TC_SKIP=40
run ICNNM_TC_SKIP=24
run ICNNM_TC_SKIP=32
run ICNNM_TC_SKIP=8
run ICNNM_TC_SKIP=1
run ICNNM_TC_SKIP=2
run ICNNM_TC_SKIP=3
timeout 120 python tools/gram_profile.py --config 2
timeout 120 python tools/gram_profile.py --config 3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:gram --log-file gpurun_out/s7_gram_launches.csv python tools/gram_profile.py --config 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:gram --log-file gpurun_out/s7_gram_launches3.csv python tools/gram_profile.py --config 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gram_lags -c 2 -o gpurun_out/s7_gram_full -f python tools/gram_profile.py --config 2 > gpurun_out/s7_gram_ncu.log 2>&1
