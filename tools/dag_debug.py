"""Development aid: compare the DAG factorization against the level path front by front."""
import os, sys
import numpy as np
sys.path.insert(0, ".")
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2_riga"
import paper_2112_14064_b200 as rq
P = rq.baseline_config(cfg)
o = rq.nested_dissection_order(P)
os.environ["RQB_FACTOR"] = "dag"
fa = rq.lu_factorize((P.rowptr, P.col, P.q_values(-0.5)), o)
os.environ["RQB_FACTOR"] = "level"
fb = rq.lu_factorize((P.rowptr, P.col, P.q_values(-0.5)), o)
print("dag", fa.info(), "level", fb.info())
nbad = 0
for fr in range(len(o.nf)):
    Fa, pa, _ = fa.front(fr)
    Fb, pb, _ = fb.front(fr)
    nf = int(o.nf[fr])
    d = np.abs(Fa[:nf, :nf] - Fb[:nf, :nf])
    m = d.max() / max(np.abs(Fb[:nf, :nf]).max(), 1e-300)
    if m > 1e-9 or not np.array_equal(pa, pb):
        bad = np.argwhere(d > 1e-9 * np.abs(Fb[:nf, :nf]).max())
        print(f"front {fr} nf={nf} npiv={o.npiv[fr]} lev={o.level[fr]} parent={o.parent[fr]} "
              f"relerr={m:.2e} ipiv_eq={np.array_equal(pa, pb)} nbad={len(bad)} "
              f"rows[{bad[:,0].min() if len(bad) else -1}..{bad[:,0].max() if len(bad) else -1}] "
              f"cols[{bad[:,1].min() if len(bad) else -1}..{bad[:,1].max() if len(bad) else -1}]", flush=True)
        nbad += 1
        if nbad > 25:
            break
print("done, bad fronts:", nbad)
