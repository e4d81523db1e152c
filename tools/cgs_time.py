"""Block CGS kernel rates (development aid): gemm_t (H = V^T R) and gemm_n
(R -= V H) over k basis vectors for block widths 1..8, L2 scrubbed."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_14064_b200 as rq  # noqa: E402
from paper_2112_14064_b200 import _lib  # noqa: E402

P = rq.baseline_config(sys.argv[1] if len(sys.argv) > 1 else "cfg4_riga")
op = rq.build_operator(P, -0.5)
hbm = 6454.9
out = {}
for k in (64, 160):
    for w in (1, 4, 8):
        for what, name in ((11, "gemm_t"), (12, "gemm_n")):
            ms = C.c_double()
            _lib.check(_lib.lib.rq_operator_time(op._h, what | 0x100, 10, k | (w << 16), C.byref(ms)))
            b = 8.0 * 2 * P.n * (k + (w if what == 11 else 2 * w))
            out[f"{name}_k{k}_w{w}"] = {"ms": round(ms.value, 4), "gbs": round(b / (ms.value * 1e6), 1),
                                        "frac": round(b / (ms.value * 1e6) / hbm, 3)}
    for what, name in ((3, "gemv_t"), (4, "gemv_n")):
        ms = C.c_double()
        _lib.check(_lib.lib.rq_operator_time(op._h, what | 0x100, 10, k, C.byref(ms)))
        b = 8.0 * 2 * P.n * k
        out[f"{name}_k{k}"] = {"ms": round(ms.value, 4), "gbs": round(b / (ms.value * 1e6), 1)}
print(json.dumps(out, indent=0))
