"""A few multi-RHS solves on one config (profiling target for ncu)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_14064_b200 as rq  # noqa: E402
from paper_2112_14064_b200 import _lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4_riga"
ks = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,4,8").split(",")]
P = rq.baseline_config(name)
op = rq.build_operator(P, -0.5)
ms = C.c_double()
for k in ks:
    _lib.check(_lib.lib.rq_operator_time(op._h, 10 | 0x100, 2, k, C.byref(ms)))
_lib.check(_lib.lib.rq_operator_time(op._h, 1 | 0x100, 2, 0, C.byref(ms)))
print("done")
