"""Factorization device time per config (development aid)."""
import sys
sys.path.insert(0, ".")
import paper_2112_14064_b200 as rq
for cfg in sys.argv[1:]:
    P = rq.baseline_config(cfg)
    o = rq.nested_dissection_order(P)
    f = rq.lu_factorize((P.rowptr, P.col, P.q_values(-0.5)), o)
    best = 1e9
    for _ in range(5):
        f.refactor(P.q_values(-0.5))
        best = min(best, f.info()["factor_ms"])
    print(f"{cfg}: factor {best:.3f} ms {o.stats['flops_lu'] / best / 1e6:.1f} GF/s", flush=True)
