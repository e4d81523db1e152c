"""Block Krylov-Schur trace on one config (development aid): per-cycle stderr
lines (RQB_EIGS_TRACE) and the final info, for a list of block sizes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("RQB_EIGS_TRACE", "1")
import paper_2112_14064_b200 as rq  # noqa: E402

name = sys.argv[1]
nev = int(sys.argv[2])
blocks = [int(x) for x in sys.argv[3].split(",")]
maxr = int(sys.argv[4]) if len(sys.argv) > 4 else 100
P = rq.baseline_config(name)
op = rq.build_operator(P, -0.5)
for bs in blocks:
    for rep in range(2):
        t = time.time()
        pairs = op.solve_quadratic(nev, eps=1e-10, block=bs, max_restarts=maxr, raise_partial=False)
        dt = time.time() - t
        i = op.last_info
        print(f"{name} block {bs} run {rep}: {dt*1e3:.1f} ms, cycles {i['restarts']}, nconv {i['nconv']}, "
              f"n_fb {i['n_fb']}, resid max {max(p.residual for p in pairs):.2e}", flush=True)
