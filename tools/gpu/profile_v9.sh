timeout 500 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo BENCH $?
for c in cfg4_riga cfg4_iga; do timeout 200 python tools/updcb_bench.py $c >> gpurun_out/updcb.jsonl; done
ncu --set full --clock-control none -k regex:updcb_bench -s 1 -c 1 -o gpurun_out/ncu_updcb_cfg4_riga_v9 python tools/updcb_bench.py cfg4_riga 2 > /dev/null 2>&1; echo NCU1 $?
ncu --set full --clock-control none -k regex:factor_dag -c 1 -o gpurun_out/ncu_fd_cfg4_v9 python tools/factor_once.py cfg4_riga > /dev/null 2>&1; echo NCU2 $?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v9.csv python bench.py --steps 2 --warmup 3 --cpu-sample-s 0 --nev-runs 1 --large '' > gpurun_out/ncu_bench.log 2>&1; echo L $?
