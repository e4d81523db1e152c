ncu --set full --import-source on --clock-control none -k regex:factor_dag -c 1 -o gpurun_out/ncu_fd_cfg2_v12 python tools/factor_once.py cfg2_riga > /dev/null 2>&1; echo N1 $?
ncu --set full --clock-control none -k regex:gemv_t_part -s 2 -c 1 -o gpurun_out/ncu_gemvt_cfg4_v12 python tools/krylov_prof.py cfg4_riga > /dev/null 2>&1; echo N2 $?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v12.csv python bench.py --steps 2 --warmup 3 --cpu-sample-s 0 --nev-runs 1 --large '' > gpurun_out/ncu_bench.log 2>&1; echo L $?
