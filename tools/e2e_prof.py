"""End-to-end profile (development aid): build_operator from a host pencil
(symbolic + uploads + factor; RQB_SETUP_TRACE=1 prints the phases), the
first and a warm solve_quadratic, twice."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_14064_b200 as rq  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4_riga"
P = rq.baseline_config(cfg)
PH = rq.QuadraticPencil(**{k: getattr(P, k) for k in ("kind", "degree", "elems", "levels", "n_full", "n", "rowptr",
                                                       "col", "K", "C", "M", "box", "free_to_full")})
for rep in range(2):
    t0 = time.perf_counter()
    op = rq.build_operator(PH, -0.5)
    t1 = time.perf_counter()
    op.solve_quadratic(100, eps=1e-10, seed=0, max_restarts=100, raise_partial=False, block=4)
    t2 = time.perf_counter()
    op.solve_quadratic(100, eps=1e-10, seed=0, max_restarts=100, raise_partial=False, block=4)
    t3 = time.perf_counter()
    print(f"build {1e3*(t1-t0):.1f} ms, first solve {1e3*(t2-t1):.1f} ms, warm solve {1e3*(t3-t2):.1f} ms",
          flush=True)
    del op
