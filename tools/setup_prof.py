import time, os
os.environ["RQB_SETUP_TRACE"]="1"
import paper_2112_14064_b200 as rq
for nm in ["cfg4_riga"]:
    t=time.perf_counter(); R = rq.baseline_config(nm, device=True, resident=True); print("assemble", (time.perf_counter()-t)*1e3, flush=True)
    t=time.perf_counter(); o = rq.nested_dissection_order(R); print("nd", (time.perf_counter()-t)*1e3, flush=True)
    t=time.perf_counter(); op = rq.build_operator(R, -0.5, o); print("build_operator resident", (time.perf_counter()-t)*1e3, flush=True)
    del op
    t=time.perf_counter(); op = rq.build_operator(R, -0.5, o); print("build_operator resident again", (time.perf_counter()-t)*1e3, flush=True)
