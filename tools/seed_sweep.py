"""Seed sweep of the Krylov-Schur time to nev on one config (development aid):
for each block size and start-vector seed, cycles / solves / wall ms (second
call on a warm operator) and the max residual. Usage:
  python tools/seed_sweep.py cfg4_riga 100 4,1 0-11"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_14064_b200 as rq  # noqa: E402

name, nev = sys.argv[1], int(sys.argv[2])
blocks = [int(x) for x in sys.argv[3].split(",")]
a, b = (int(x) for x in sys.argv[4].split("-"))
P = rq.baseline_config(name)
op = rq.build_operator(P, -0.5)
op.solve_quadratic(nev, eps=1e-10, block=blocks[0], max_restarts=100, raise_partial=False)  # warm-up
for bs in blocks:
    ms, cyc = [], []
    for seed in range(a, b + 1):
        t = time.time()
        pairs = op.solve_quadratic(nev, eps=1e-10, seed=seed, block=bs, max_restarts=100, raise_partial=False)
        dt = (time.time() - t) * 1e3
        i = op.last_info
        ms.append(dt)
        cyc.append(i["restarts"])
        print(f"{name} block {bs} seed {seed}: {dt:.1f} ms, cycles {i['restarts']}, nconv {i['nconv']}, "
              f"n_fb {i['n_fb']}, resid max {max(p.residual for p in pairs):.2e}", flush=True)
    print(f"== block {bs}: median {statistics.median(ms):.1f} ms, mean {statistics.mean(ms):.1f}, "
          f"cycles median {statistics.median(cyc)}", flush=True)
