"""One factorization + two solves of a config (ncu launch-list target; development aid)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2112_14064_b200 as rq
P = rq.baseline_config(sys.argv[1] if len(sys.argv) > 1 else "cfg2_riga")
o = rq.nested_dissection_order(P)
f = rq.lu_factorize((P.rowptr, P.col, P.q_values(-0.5)), o)
b = np.random.default_rng(0).standard_normal(P.n)
for _ in range(2):
    x = f.solve(b)
print(f.info())
