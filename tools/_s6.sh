run() { echo "=== $*"; env "$@" python tools/with_ab_lib.py tools/tc_counters.py --config ${CFG:-4} --iters 20 2>&1 | head -3 | sed -e 's/np.float64(//g; s/)//g'; }
run A=0
run ICNNM_TC_WARR=0
run ICNNM_DET=0
run ICNNM_DET=0 ICNNM_TC_WARR=0
CFG=2 run A=0
CFG=2 run ICNNM_TC_WARR=0
CFG=2 run ICNNM_DET=0
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
bash tools/_s5.sh
