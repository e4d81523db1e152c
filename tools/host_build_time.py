"""build_operator from host arrays in a warm process (development aid):
python tools/host_build_time.py cfg4_riga"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_14064_b200 as rq
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4_riga"
P = rq.baseline_config(cfg)
o = rq.nested_dissection_order(P)
f = rq.lu_factorize((P.rowptr, P.col, P.q_values(-0.5)), o)  # warm the process
del f
for rep in range(3):
    PH = rq.QuadraticPencil(**{k: getattr(P, k) for k in ("kind", "degree", "elems", "levels", "n_full", "n", "rowptr",
                                                           "col", "K", "C", "M", "box", "free_to_full")})
    t0 = time.perf_counter()
    op = rq.build_operator(PH, -0.5, o)
    print(f"rep {rep}: build from host {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    del op
