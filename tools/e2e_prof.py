"""Where the host-to-eigenpairs time goes at one config (development aid)."""
import os, sys, time
sys.path.insert(0, ".")
os.environ.setdefault("RQB_SETUP_TRACE", "1")
import paper_2112_14064_b200 as rq
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2_riga"
nev = int(sys.argv[2]) if len(sys.argv) > 2 else 20
P = rq.baseline_config(cfg)
t = time.perf_counter(); o = rq.nested_dissection_order(P); print("nd", (time.perf_counter() - t) * 1e3, flush=True)
for rep in range(2):
    t = time.perf_counter(); op = rq.build_operator(P, -0.5, o); t1 = time.perf_counter()
    op.solve_quadratic(nev, eps=1e-10, seed=0); t2 = time.perf_counter()
    op.solve_quadratic(nev, eps=1e-10, seed=0); t3 = time.perf_counter()
    print(f"rep {rep}: build_operator {(t1-t)*1e3:.1f} ms, first solve {(t2-t1)*1e3:.1f} ms, second solve {(t3-t2)*1e3:.1f} ms",
          op.last_info, flush=True)
    del op
