"""Spread of the eigensolve over start-vector seeds (development aid): the
degenerate BASELINE cluster makes the Krylov-Schur cycle count sensitive to
rounding, so time to nev is reported as min / median / max over seeds."""
import sys, json
import numpy as np
sys.path.insert(0, ".")
import paper_2112_14064_b200 as rq
NEV = {"cfg1": 10, "cfg2_riga": 20, "cfg2_iga": 20, "cfg3_riga": 50, "cfg3_iga": 50, "cfg4_riga": 100, "cfg4_iga": 100}
cfg = sys.argv[1]
seeds = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 2, 3, 4]
P = rq.baseline_config(cfg)
op = rq.build_operator(P, -0.5)
op.solve_quadratic(NEV[cfg], max_restarts=1000, raise_partial=False)  # warm-up
rows = []
for s in seeds:
    pairs = op.solve_quadratic(NEV[cfg], seed=s, max_restarts=1000, raise_partial=False)
    i = op.last_info
    rows.append((s, i["t_total_ms"], i["restarts"], i["n_fb"], i["nconv"], max(p.residual for p in pairs)))
    print(f"  seed {s}: {i['t_total_ms']:.1f} ms cycles {i['restarts']} n_fb {i['n_fb']} nconv {i['nconv']} resmax {rows[-1][-1]:.2e}", flush=True)
t = np.array([r[1] for r in rows])
print(json.dumps({"config": cfg, "nev": NEV[cfg], "seeds": seeds, "time_ms_min": round(t.min(), 1),
                  "time_ms_median": round(float(np.median(t)), 1), "time_ms_max": round(t.max(), 1),
                  "cycles": [r[2] for r in rows], "n_fb": [r[3] for r in rows]}))
