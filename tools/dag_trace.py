"""Timeline of one traced factorization (development aid): runs
rq_factor_dag_profile with RQB_DAG_TRACE and prints per-level windows and the
front-by-front critical path."""
import os, sys, ctypes as C
import numpy as np
sys.path.insert(0, ".")
out = "gpurun_out/dag_trace.bin"
os.environ["RQB_DAG_TRACE"] = out
import paper_2112_14064_b200 as rq
from paper_2112_14064_b200 import _lib, sparsela as sl
cfg = sys.argv[1]
P = rq.baseline_config(cfg)
o = rq.nested_dissection_order(P)
f = rq.lu_factorize((P.rowptr, P.col, P.q_values(-0.5)), o)
f.refactor(P.q_values(-0.5))
prof = np.zeros(24)
_lib.check(_lib.lib.rq_factor_dag_profile(f._h, prof))
raw = open(out, "rb").read()
nt = int(np.frombuffer(raw, np.int32, 1, 0)[0])
tk = np.frombuffer(raw, np.dtype([("front", "<i4"), ("type", "<i2"), ("step", "<i2"), ("a", "<i4"), ("b", "<i4")]), nt, 4)
allt = np.frombuffer(raw, np.uint64, 4 * nt, 4 + 16 * nt).astype(np.int64)
tr = allt[:2 * nt].reshape(-1, 2).copy()
ph = allt[2 * nt:].reshape(-1, 2).copy()  # {work done, fence done}
valid = (tr[:, 0] > 0) & (tr[:, 1] > 0)
t00 = tr[valid, 0].min()
tr = np.where(valid[:, None], tr - t00, 0)
ph = np.where(valid[:, None], ph - t00, 0)
print(f"untraced tasks: {(~valid).sum()} of {nt}; types", np.unique(tk['type'][~valid]))
names = ["SMALL", "ASM", "DIAG", "ROWS", "COLS", "UPD", "UPDCB", "UPDB"]
nfr = len(o.parent)
fs = np.full(nfr, 1 << 62); fe = np.zeros(nfr, np.int64)
np.minimum.at(fs, tk["front"][valid], tr[valid, 0]); np.maximum.at(fe, tk["front"][valid], tr[valid, 1])
print(f"{cfg}: span {tr[:,1].max()/1e3:.1f} us, tasks {nt}")
lv = o.level
for L in sorted(set(lv.tolist())):
    m = lv == L
    print(f"  level {L:2d} fronts {m.sum():5d} nf {o.nf[m].min()}-{o.nf[m].max()} npiv {o.npiv[m].min()}-{o.npiv[m].max()} start {fs[m].min()/1e3:8.1f} end {fe[m].max()/1e3:8.1f} us  mean front span {(fe[m]-fs[m]).mean()/1e3:7.1f} us")
# critical path: from the root back through the latest-finishing child
child_end = {}
for c in range(nfr):
    p = o.parent[c]
    if p >= 0 and fe[c] > child_end.get(p, (-1, -1))[0]:
        child_end[p] = (fe[c], c)
f_ = int(np.argmax(fe))
print("  critical chain (front nf npiv: ready -> start -> end, us):")
while True:
    ready = child_end.get(f_, (0, -1))[0]
    ty = tk["type"][tk["front"] == f_]
    cnts = {names[t]: int((ty == t).sum()) for t in range(8) if (ty == t).sum()}
    print(f"    front {f_:5d} nf {o.nf[f_]:5d} npiv {o.npiv[f_]:5d} level {lv[f_]:2d}: ready {ready/1e3:8.1f} start {fs[f_]/1e3:8.1f} end {fe[f_]/1e3:8.1f}  {cnts}")
    if f_ not in child_end: break
    f_ = child_end[f_][1]
if len(sys.argv) > 2:  # task list of one front
    ff = int(sys.argv[2])
    idx = np.nonzero(tk["front"] == ff)[0]
    idx = idx[np.argsort(tr[idx, 0])]
    for i in idx[:200]:
        print(f"     {names[tk['type'][i]]:5s} s{tk['step'][i]:3d} a{tk['a'][i]:3d} b{tk['b'][i]:3d}  {tr[i,0]/1e3:8.2f} -> {tr[i,1]/1e3:8.2f}  ({(tr[i,1]-tr[i,0])/1e3:6.2f})  work {(ph[i,0]-tr[i,0])/1e3:6.2f} fence {(ph[i,1]-ph[i,0])/1e3:6.2f} succ {(tr[i,1]-ph[i,1])/1e3:6.2f}")
# busy-CTA profile over time (20 bins): concurrent tasks, and the share of
# tasks by type per bin
span = tr[:, 1].max()
bins = np.linspace(0, span, 21)
print("  busy profile (bin: active task-us / bin width, by type):")
for b0, b1 in zip(bins[:-1], bins[1:]):
    ov = np.clip(np.minimum(tr[:, 1], b1) - np.maximum(tr[:, 0], b0), 0, None)
    tot = ov.sum() / (b1 - b0)
    by = {names[t]: round(float(ov[tk["type"] == t].sum() / (b1 - b0)), 1) for t in range(8)}
    print(f"   {b0/1e3:7.1f}-{b1/1e3:7.1f} us: {tot:6.1f}  {by}")
# per-type phase split on the top fronts (levels >= 11): work / fence / successor release, us
top = np.isin(tk["front"], np.nonzero(o.level >= 11)[0]) & valid
print("  phase split on levels >= 11 (mean us: total, work, fence, succ):")
for t in range(8):
    m_ = top & (tk["type"] == t)
    if m_.sum() == 0:
        continue
    tot_ = (tr[m_, 1] - tr[m_, 0]).mean() / 1e3
    wk = (ph[m_, 0] - tr[m_, 0]).mean() / 1e3
    fe_ = (ph[m_, 1] - ph[m_, 0]).mean() / 1e3
    sc = (tr[m_, 1] - ph[m_, 1]).mean() / 1e3
    print(f"   {names[t]:5s} n {m_.sum():6d}  {tot_:7.2f} {wk:7.2f} {fe_:7.2f} {sc:7.2f}")
# gaps on the root's panel chain: DIAG(s) start - end of the latest predecessor-type task of step s-1
root = int(np.argmax(o.level))
d = np.nonzero((tk["front"] == root) & (tk["type"] == 2) & valid)[0]
d = d[np.argsort(tk["step"][d])]
print("  root DIAG starts (us) and step-to-step deltas:", [round(float(tr[i, 0]) / 1e3, 1) for i in d[:6]],
      [round(float(tr[d[k + 1], 0] - tr[d[k], 0]) / 1e3, 1) for k in range(min(12, len(d) - 1))])
