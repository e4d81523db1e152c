"""Trace the two triangular sweeps item by item (development aid).
Runs one solve with RQB_SOLVE_TRACE and prints phase sums and the busy profile."""
import os, sys, ctypes as C
import numpy as np
sys.path.insert(0, ".")
out = "gpurun_out/solve_trace.bin"
if os.path.exists(out):
    os.remove(out)
os.environ["RQB_SOLVE_TRACE"] = out
import paper_2112_14064_b200 as rq
from paper_2112_14064_b200 import _lib, sparsela as sl
cfg = sys.argv[1]
P = rq.baseline_config(cfg)
op = rq.build_operator(P, -0.5)
o = sl.Ordering(P.n, P.box, P.elems)
ms = C.c_double()
_lib.check(_lib.lib.rq_operator_time(op._h, 1, 3, 0, C.byref(ms)))
raw = open(out, "rb").read()
recs = []
pos = 0
while pos < len(raw):
    nf_, nb_ = np.frombuffer(raw, np.int32, 2, pos); pos += 8
    cnt = 8 * (nf_ + nb_)
    t = np.frombuffer(raw, np.uint64, cnt, pos).reshape(-1, 8).astype(np.int64); pos += 8 * cnt
    recs.append((nf_, nb_, t))
nf_, nb_, t = recs[-1]
import pickle
pickle.dump((nf_, nb_, t, o.parent, o.npiv, o.nf, o.level), open(f"gpurun_out/solve_trace_{cfg}.pkl", "wb"))
npb = (o.npiv + 63) // 64; ncbb = (o.nf - o.npiv + 63) // 64
ffront = np.repeat(np.arange(len(npb)), npb + ncbb)
for name, T in (("fwd", t[:nf_]), ("bwd", t[nf_:])):
    t0 = T[:, 0].min()
    T = T.copy(); T[:, :4] -= t0
    span = T[:, 3].max()
    g = (T[:, 1] - T[:, 0]); l = (T[:, 2] - T[:, 1]); e = (T[:, 3] - T[:, 2])
    w = T[:, 5]
    busy = (T[:, 3] - T[:, 0]).sum()
    print(f"   waited {w.sum()/1e3:.0f} us of loop; busy-CTA time {busy/1e3:.0f} us over span*grid {span*444/1e3:.0f} us")
    print(f"{name}: items {len(T)} span {span/1e3:.1f} us  sum gather {g.sum()/1e3:.0f} loop {l.sum()/1e3:.0f} tail {e.sum()/1e3:.0f} us; "
          f"mean per item gather {g.mean():.0f} loop {l.mean():.0f} tail {e.mean():.0f} ns")
    # concurrency profile: number of active items over time (10 bins)
    bins = np.linspace(0, span, 11)
    act = [((T[:, 0] < b1) & (T[:, 3] > b0)).sum() for b0, b1 in zip(bins[:-1], bins[1:])]
    print("   active items per span decile:", act)
    # pop gaps: per SM sort by start; gap = start - previous end on same SM (approx CTA)
    first = T[:, 0].argsort()[:5]
    print("   first starts (ns):", T[first, 0].tolist(), " last ends:", np.sort(T[:, 3])[-5:].tolist())
