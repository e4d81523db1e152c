"""Multi-RHS sweep timing (development aid): device ms of the single-vector
sweeps and of the multi-RHS sweeps for 1..8 right-hand sides, L2 scrubbed,
with the effective per-vector bandwidth against the trisolve algorithmic bytes."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_14064_b200 as rq  # noqa: E402
from paper_2112_14064_b200 import _lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4_riga"
P = rq.baseline_config(name)
op = rq.build_operator(P, -0.5)
st = op.ordering.stats


def t(what, param, iters=10):
    ms = C.c_double()
    _lib.check(_lib.lib.rq_operator_time(op._h, what | 0x100, iters, param, C.byref(ms)))
    return ms.value


out = {"config": name, "trisolve_bytes": st.get("trisolve_bytes"), "single_solve_ms": t(1, 0), "single_apply_ms": t(0, 0)}
for k in (1, 2, 4, 8):
    out[f"msolve{k}_ms"] = t(10, k)
    out[f"apply_block{k}_ms"] = t(9, k)
print(json.dumps(out))
