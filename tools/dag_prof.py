"""Task-level profile of the persistent factorization (development aid)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2112_14064_b200 as rq
from paper_2112_14064_b200 import _lib
for cfg in sys.argv[1:]:
    P = rq.baseline_config(cfg)
    o = rq.nested_dissection_order(P)
    f = rq.lu_factorize((P.rowptr, P.col, P.q_values(-0.5)), o)
    for _ in range(3):
        f.refactor(P.q_values(-0.5))
    out = np.zeros(24)
    _lib.check(_lib.lib.rq_factor_dag_profile(f._h, out))
    info = f.info()
    names = ["SMALL", "ASM", "DIAG", "ROWS", "COLS", "UPD"]
    print(f"{cfg}: factor {info['factor_ms']:.3f} ms {info['gflops']:.1f} GF/s grid {int(out[18])} tasks {int(out[19])} popwait {out[20]:.2f} ms"
          f" flops {o.stats['flops_lu']:.3e} max_front {o.stats['max_front']}")
    for t, nm in enumerate(names):
        busy, wait, cnt = out[3 * t:3 * t + 3]
        if cnt:
            print(f"   {nm:6s} n={int(cnt):7d} busy={busy:9.3f} ms (avg {busy / cnt * 1e3:8.2f} us)")
    if out[23]:
        print(f"   UPDCB  n={int(out[23]):7d} busy={out[21]:9.3f} ms (avg {out[21] / out[23] * 1e3:8.2f} us)")
