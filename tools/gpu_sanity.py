"""Quick device sanity run (development aid): factor/solve/apply/eigs vs the oracle."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import oracle
import paper_2112_14064_b200 as rq

for cfg in sys.argv[1:] or ["cfg1"]:
    p = rq.baseline_config(cfg)
    t = time.time()
    op = rq.build_operator(p, -0.5)
    print(cfg, "n", p.n, "build s", round(time.time() - t, 3), op.factor_info(), flush=True)
    of = oracle.Factor(p.n, p.rowptr, p.col, p.q_values(-0.5), p.box, p.elems)
    f = op.ordering
    b = np.random.default_rng(1).standard_normal(p.n)
    fac = rq.lu_factorize((p.rowptr, p.col, p.q_values(-0.5)), f)
    x = fac.solve(b)
    xo = of.solve(b).real
    print(" solve rel err", np.max(np.abs(x - xo)) / np.max(np.abs(xo)), "info", fac.info(), flush=True)
    v = np.random.default_rng(2).uniform(-1, 1, 2 * p.n)
    r = op.apply(v)
    E = oracle.Eig(p, -0.5)
    ro = E.apply(v).real
    print(" apply rel err", np.max(np.abs(r - ro)) / np.max(np.abs(ro)), flush=True)
    nev = {"cfg1": 10}.get(cfg, 20)
    t = time.time()
    pairs = op.solve_quadratic(nev, raise_partial=False)
    print(" eigs s", round(time.time() - t, 3), op.last_info, flush=True)
    print(" lam", [complex(round(q.lam.real, 10), round(q.lam.imag, 10)) for q in pairs[:4]], "res max", max(q.residual for q in pairs))
