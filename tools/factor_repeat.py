"""Repeat a factorization many times (development aid: intermittent stalls)."""
import sys
sys.path.insert(0, ".")
import paper_2112_14064_b200 as rq
cfg, reps = sys.argv[1], int(sys.argv[2])
P = rq.baseline_config(cfg)
o = rq.nested_dissection_order(P)
f = rq.lu_factorize((P.rowptr, P.col, P.q_values(-0.5)), o)
bad = 0
for i in range(reps):
    try:
        f.refactor(P.q_values(-0.5))
    except Exception as e:  # noqa: BLE001
        bad += 1
        print("rep", i, "error:", str(e)[:400], flush=True)
        if bad > 2:
            break
print(cfg, "reps", reps, "errors", bad, "last ms", f.info()["factor_ms"], "swaps", f.info()["swaps"])
