timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo TESTS $?; tail -2 gpurun_out/gpu_tests.log
for c in cfg2_riga cfg4_riga; do timeout 300 python tools/solve_prof.py $c 2>&1 | tail -1; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/factor_once.py ${1:-cfg2_riga} > gpurun_out/ncu_fo.csv 2>&1; grep -E "gpu__time" gpurun_out/ncu_fo.csv | awk -F'","' '{print $5, $NF}' | cut -c1-40,200- | sed 's/(.*)//' 
