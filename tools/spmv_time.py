"""CSR product rates on one config (development aid): the fused C/M operator
SpMV, the block operator SpMM and the block M-SpMM at widths 4 / 8, L2
scrubbed; run once per RQB_SPMV version to compare."""
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
out = {"version": os.environ.get("RQB_SPMV", "2")}


def t(what, param):
    ms = C.c_double()
    _lib.check(_lib.lib.rq_operator_time(op._h, what | 0x100, 20, param, C.byref(ms)))
    return ms.value


pat = 12.0 * P.nnz + 8.0 * (P.n + 1)  # col + one value array + rowptr
for name, what, w, b in (("spmv_op", 2, 1, pat + 8.0 * P.nnz + 24.0 * P.n),
                         ("spmm_op_4", 13, 4, pat + 8.0 * P.nnz + 8.0 * P.n * (2 * 4 + 4)),
                         ("spmm_op_8", 13, 8, pat + 8.0 * P.nnz + 8.0 * P.n * (2 * 8 + 8)),
                         ("spmm_m_4", 14, 4, pat + 8.0 * P.n * (4 + 4)),
                         ("spmm_m_8", 14, 8, pat + 8.0 * P.n * (8 + 8))):
    ms = t(what, w)
    out[name] = {"ms": round(ms, 4), "gbs": round(b / (ms * 1e6), 1), "frac": round(b / (ms * 1e6) / hbm, 3)}
print(json.dumps(out))
