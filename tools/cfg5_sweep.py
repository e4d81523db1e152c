"""BASELINE configs[4] (cfg5): H(curl) 256^2 factorization sweep p = 2..5, IGA vs
rIGA (front-size distribution and GFLOP/s per tree level), and at p = 3 rIGA the
full eigensolve for nev = 10, 50, 200 (phase split). One JSON line per run.
usage: python tools/cfg5_sweep.py [--part 1|2|both]"""
import json, os, sys
import numpy as np
sys.path.insert(0, ".")
trace = "/tmp/cfg5_dag_trace.bin"
os.environ["RQB_DAG_TRACE"] = trace
import paper_2112_14064_b200 as rq
from paper_2112_14064_b200 import _lib

part = sys.argv[sys.argv.index("--part") + 1] if "--part" in sys.argv else "both"
SIGMA = -0.5
if part in ("1", "both"):
    for p in (2, 3, 4, 5):
        for kind in ("iga", "riga"):
            name = f"cfg5_p{p}_{kind}"
            P = rq.baseline_config(name)
            o = rq.nested_dissection_order(P)
            f = rq.lu_factorize((P.rowptr, P.col, P.q_values(SIGMA)), o)
            best = 1e9
            for _ in range(3):
                f.refactor(P.q_values(SIGMA))
                best = min(best, f.info()["factor_ms"])
            # per-level flops and the level's busy window in one traced factorization
            prof = np.zeros(24)
            _lib.check(_lib.lib.rq_factor_dag_profile(f._h, prof))
            raw = open(trace, "rb").read()
            nt = int(np.frombuffer(raw, np.int32, 1, 0)[0])
            tk = np.frombuffer(raw, np.dtype([("front", "<i4"), ("type", "<i2"), ("step", "<i2"), ("a", "<i4"), ("b", "<i4")]), nt, 4)
            tr = np.frombuffer(raw, np.uint64, 2 * nt, 4 + 16 * nt).reshape(-1, 2).astype(np.int64)
            tr -= tr[:, 0].min()
            nf, npv = o.nf.astype(np.float64), o.npiv.astype(np.float64)
            # F_LU per front: sum_k (nf-k-1) + 2 (nf-k-1)^2
            fl = np.zeros(len(nf))
            for i in range(len(nf)):
                r = nf[i] - np.arange(npv[i]) - 1.0
                fl[i] = (r + 2 * r * r).sum()
            lv = o.level
            levels = []
            for L in sorted(set(lv.tolist())):
                m = lv[tk["front"]] == L
                t0, t1 = tr[m, 0].min(), tr[m, 1].max()
                busy = (tr[m, 1] - tr[m, 0]).sum()
                fL = fl[lv == L].sum()
                levels.append({"level": L, "fronts": int((lv == L).sum()), "nf_max": int(nf[lv == L].max()),
                               "gflop": round(fL / 1e9, 4), "window_ms": round((t1 - t0) / 1e6, 4),
                               "gflops_window": round(fL / max(t1 - t0, 1), 2),
                               "gflops_per_busy_cta": round(fL / max(busy, 1), 2)})
            hist = np.histogram(o.nf, bins=[0, 64, 128, 256, 512, 1024, 2048, 4096, 8192])[0].tolist()
            line = {"config": name, "n": P.n, "nnz": P.nnz, "nnz_l": int(o.stats["nnz_l"]), "flops_lu": o.stats["flops_lu"],
                    "max_front": int(o.stats["max_front"]), "factor_ms": round(best, 3),
                    "gflops": round(o.stats["flops_lu"] / best / 1e6, 1),
                    "front_size_hist": {"edges": [0, 64, 128, 256, 512, 1024, 2048, 4096, 8192], "counts": hist},
                    "levels": levels}
            print(json.dumps(line), flush=True)
if part in ("2", "both"):
    P = rq.baseline_config("cfg5_p3_riga")
    op = rq.build_operator(P, SIGMA)
    for nev in (10, 50, 200):
        op.solve_quadratic(nev, max_restarts=1000, raise_partial=False, profile=True)  # warm (graphs, cuBLAS)
        pairs = op.solve_quadratic(nev, max_restarts=1000, raise_partial=False, profile=True)
        i = op.last_info
        line = {"config": "cfg5_p3_riga", "nev": nev, "m": 2 * nev + 1, "nconv": i["nconv"],
                "time_ms": round(i["t_total_ms"], 1), "solve_ms": round(i["t_solve_ms"], 1),
                "orth_ms": round(i["t_orth_ms"], 1), "ritz_ms": round(i["t_ritz_ms"], 1),
                "check_ms": round(i["t_check_ms"], 1), "restart_ms": round(i["t_restart_ms"], 1),
                "cycles": i["restarts"], "n_fb": i["n_fb"], "residual_max": max(p.residual for p in pairs),
                "note": "profile=True (per-phase CUDA events, no graphs): phase split, not the fastest wall time"}
        print(json.dumps(line), flush=True)
