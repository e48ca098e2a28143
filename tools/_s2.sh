set -x
python tools/with_ab_lib.py tools/tc_counters.py --config 4 --iters 5 > gpurun_out/s2_cnt4.txt 2>&1
python tools/with_ab_lib.py tools/tc_counters.py --config 2 --iters 5 > gpurun_out/s2_cnt2.txt 2>&1
python bench.py --config 2 --no-cpu-baseline > gpurun_out/s2_bench2.json 2> gpurun_out/s2_bench2.err
python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2_bench3.json 2> gpurun_out/s2_bench3.err
python tools/profile_step.py --config 4 --iters 3 > gpurun_out/s2_ps4.txt 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:icnnm_tc -c 6 -o gpurun_out/s2_full4 -f python tools/profile_step.py --config 4 --iters 3 > gpurun_out/s2_ncu4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s2_launches4.csv python bench.py --batch 2 --iters 40 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s2_ncul.log 2>&1
