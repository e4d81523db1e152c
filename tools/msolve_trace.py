"""Per-level timeline of the multi-RHS sweeps (development aid): one traced
multi-RHS solve (RQB_MSOLVE_TRACE) of `k` right-hand sides on a config."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
out = "gpurun_out/msolve_trace.bin"
os.environ["RQB_MSOLVE_TRACE"] = out
import paper_2112_14064_b200 as rq  # noqa: E402
from paper_2112_14064_b200 import _lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4_riga"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
whole_min = int(os.environ.get("RQB_MWHOLE_MIN", "128"))
P = rq.baseline_config(cfg)
op = rq.build_operator(P, -0.5)
o = op.ordering
ms = C.c_double()
_lib.check(_lib.lib.rq_operator_time(op._h, 10, 2, k, C.byref(ms)))
raw = open(out, "rb").read()
nf_, nb_ = np.frombuffer(raw, np.int32, 2, 0)
t = np.frombuffer(raw, np.uint64, 2 * (nf_ + nb_), 8).reshape(-1, 2).astype(np.int64)
npb = (o.npiv + 63) // 64
ncbb = (o.nf - o.npiv + 63) // 64
lvl_count = np.bincount(o.level)
whole = (npb <= 2) & (o.nf <= 512) & (lvl_count[o.level] >= whole_min)
fcnt = np.where(whole, 1, npb + ncbb)
ncb = o.nf - o.npiv
nck = np.where((~whole) & (npb > 0) & (ncb > 256), (ncb + 255) // 256, 0)
bcnt = np.where(npb > 0, np.where(whole, 1, npb + npb * nck), 0)
ffront = np.repeat(np.arange(len(npb)), fcnt)
bfront = np.repeat(np.arange(len(npb))[::-1], bcnt[::-1])
assert len(ffront) == nf_ and len(bfront) == nb_, (len(ffront), nf_, len(bfront), nb_)
for name, T, fr in (("fwd", t[:nf_], ffront), ("bwd", t[nf_:], bfront)):
    T = T - T[:, 0].min()
    print(f"{name}: items {len(T)} span {T[:, 1].max() / 1e3:.1f} us")
    lv = o.level[fr]
    for L in sorted(set(lv.tolist())):
        m = lv == L
        d = (T[m, 1] - T[m, 0]) / 1e3
        print(f"  level {L:2d} fronts {lvl_count[L]:5d} items {m.sum():6d} start {T[m, 0].min() / 1e3:8.1f} "
              f"end {T[m, 1].max() / 1e3:8.1f} mean item {d.mean():7.2f} us max {d.max():7.2f}")
