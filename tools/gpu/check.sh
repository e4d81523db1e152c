timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo TESTS $?; tail -3 gpurun_out/gpu_tests.log
for c in cfg2_riga cfg4_riga cfg4_iga; do timeout 300 python tools/solve_prof.py $c 2>&1 | tail -1; done
timeout 400 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo BENCH $?
python - <<'P'
import json; d=json.loads(open('gpurun_out/bench.jsonl').read().strip().splitlines()[-1])
print("value",d["value"],"ttn",d["time_to_nev_ms"],"tri",d["kernels"]["trisolve"],"large",d["large_config"]["factor"],d["large_config"]["trisolve"], "e2e", d["e2e"])
P
