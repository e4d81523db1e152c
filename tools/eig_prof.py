"""Eigensolve phase profile (development aid)."""
import sys, time
sys.path.insert(0, ".")
import paper_2112_14064_b200 as rq
NEV = {"cfg1": 10, "cfg2_riga": 20, "cfg2_iga": 20, "cfg3_riga": 50, "cfg3_iga": 50, "cfg4_riga": 100, "cfg4_iga": 100}
for cfg in sys.argv[1:]:
    t = time.perf_counter()
    P = rq.baseline_config(cfg)
    t_asm = time.perf_counter() - t
    t = time.perf_counter()
    op = rq.build_operator(P, -0.5)
    t_op = time.perf_counter() - t
    print(f"{cfg}: n {P.n} nnz {P.nnz} assemble {t_asm:.2f} s build_operator {t_op:.2f} s factor {op.factor_info()}", flush=True)
    nev = NEV[cfg]
    for prof in (False, True, False):
        t = time.perf_counter()
        pairs = op.solve_quadratic(nev, max_restarts=1000, raise_partial=False, profile=prof)
        wall = (time.perf_counter() - t) * 1e3
        i = op.last_info
        print(f"  prof={prof} wall {wall:.1f} ms total {i['t_total_ms']:.1f} solve {i['t_solve_ms']:.1f} orth {i['t_orth_ms']:.1f} "
              f"sync {i['t_sync_ms']:.1f} ritz {i['t_ritz_ms']:.1f} check {i['t_check_ms']:.1f} restart {i['t_restart_ms']:.1f} "
              f"cycles {i['restarts']} guard {i['guard_passes']} n_fb {i['n_fb']} launches {i['launches']} resmax {max(p.residual for p in pairs):.2e}", flush=True)
