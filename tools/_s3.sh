run() { echo "=== $*"; env "$@" python tools/with_ab_lib.py tools/tc_counters.py --config 4 --iters 20 2>&1 | head -3; }
run A=0
run ICNNM_TC_BTIGHT=1 ICNNM_TC_SB=16
run ICNNM_TC_BTIGHT=1 ICNNM_TC_SB=12
run ICNNM_TC_BRES=1
run ICNNM_TC_BRES=0
run ICNNM_TC_GRP=2
run ICNNM_TC_GRP=2 ICNNM_TC_BTIGHT=1 ICNNM_TC_SB=16
run ICNNM_TC_NHB=2
run ICNNM_TC_BPAIR=1
echo "=== config 2"
for e in "A=0" "ICNNM_TC_BRES=0" "ICNNM_TC_BTIGHT=1 ICNNM_TC_SB=12"; do echo "== $e"; env $e python tools/with_ab_lib.py tools/tc_counters.py --config 2 --iters 20 2>&1 | head -3; done
