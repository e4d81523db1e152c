ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v7.csv python bench.py --steps 2 --warmup 3 --cpu-sample-s 0 --nev-runs 1 --large '' > gpurun_out/ncu_bench.log 2>&1; echo L $?
for k in fwd_sweep bwd_sweep diag_inverse; do
  ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/ncu_cfg4_${k}_v7 python tools/solve_once.py cfg4_riga > /dev/null 2>&1; echo $k $?
  ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/ncu_cfg2_${k}_v7 python tools/solve_once.py cfg2_riga > /dev/null 2>&1; echo $k $?
done
