"""Large-front Schur update alone (evidence for the FP64 tensor-core target):
the factorization's own UPDCB code over every contribution-block tile of the
largest front, timed with CUDA events; run under ncu for the DMMA-pipe counters."""
import sys, json
import numpy as np
sys.path.insert(0, ".")
import paper_2112_14064_b200 as rq
from paper_2112_14064_b200 import _lib
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4_riga"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
P = rq.baseline_config(cfg)
o = rq.nested_dissection_order(P)
f = rq.lu_factorize((P.rowptr, P.col, P.q_values(-0.5)), o)
out = np.zeros(6)
_lib.check(_lib.lib.rq_factor_bench_updcb(f._h, -1, reps, out))
ms, fl = out[0], out[1]
print(json.dumps({"config": cfg, "front": int(out[2]), "K": int(out[4]), "tiles": int(out[3]), "grid": int(out[5]),
                  "ms": round(ms, 4), "gflop": round(fl / 1e9, 3), "tflops": round(fl / ms / 1e9, 2),
                  "frac_fp64_peak_37.2": round(fl / ms / 1e9 / 37.2, 3)}))
