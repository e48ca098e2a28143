run() { echo "=== $*"; env "$@" python tools/with_ab_lib.py tools/tc_counters.py --config 4 --iters 20 2>&1 | head -3 | sed -e 's/np.float64(//g; s/)//g'; }
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
