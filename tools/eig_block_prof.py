"""Block Krylov-Schur phase profile at one config (development aid):
python tools/eig_block_prof.py cfg4_riga [block] [seeds]"""
import sys, time
sys.path.insert(0, ".")
import paper_2112_14064_b200 as rq
cfg = sys.argv[1]
block = int(sys.argv[2]) if len(sys.argv) > 2 else 4
seeds = [int(s) for s in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, 1]
NEV = {"cfg2_riga": 20, "cfg3_riga": 50, "cfg4_riga": 100, "cfg4_iga": 100}
P = rq.baseline_config(cfg)
op = rq.build_operator(P, -0.5)
nev = NEV[cfg]
op.solve_quadratic(nev, max_restarts=1000, raise_partial=False, block=block)  # warm: workspace + graphs
for seed in seeds:
    for prof in (False, True):
        t = time.perf_counter()
        pairs = op.solve_quadratic(nev, seed=seed, max_restarts=1000, raise_partial=False, profile=prof, block=block)
        wall = (time.perf_counter() - t) * 1e3
        i = op.last_info
        print(f"{cfg} block {block} seed {seed} prof={prof} wall {wall:.1f} ms total {i['t_total_ms']:.1f} solve {i['t_solve_ms']:.1f} "
              f"orth {i['t_orth_ms']:.1f} sync {i['t_sync_ms']:.1f} ritz {i['t_ritz_ms']:.1f} check {i['t_check_ms']:.1f} "
              f"restart {i['t_restart_ms']:.1f} cycles {i['restarts']} n_fb {i['n_fb']} launches {i['launches']} "
              f"resmax {max(p.residual for p in pairs):.2e}", flush=True)
