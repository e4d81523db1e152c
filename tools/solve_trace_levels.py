"""Per-level timeline of a traced solve (reads gpurun_out/solve_trace_<cfg>.pkl)."""
import pickle, sys
import numpy as np
sys.path.insert(0, ".")
cfg = sys.argv[1]
nf_, nb_, t, parent, npiv, nf, level = pickle.load(open(f"gpurun_out/solve_trace_{cfg}.pkl", "rb"))
kWholeNpb, kWholeCb = int(sys.argv[2]) if len(sys.argv) > 2 else 2, 1024 - 2 * 64
npb = (npiv + 63) // 64; ncbb = (nf - npiv + 63) // 64
nfr = len(npb)
lvl_count = np.bincount(level)
whole = (npb <= kWholeNpb) & (nf - npiv <= kWholeCb)
if len(sys.argv) > 3: whole &= lvl_count[level] >= int(sys.argv[3])
fcnt = np.where(whole, 1, npb + ncbb)
ffront = np.repeat(np.arange(nfr), fcnt)
ncb = nf - npiv
nck = np.where((~whole) & (npb > 0) & (ncb > 256), (ncb + 255) // 256, 0)
bcnt = np.where(whole & (npb > 0), 1, npb + npb * nck)  # backward partial items (RQB_CB_CHUNK default 256)
bfront = np.repeat(np.arange(nfr)[::-1], bcnt[::-1])
for name, T, fr in (("fwd", t[:nf_], ffront), ("bwd", t[nf_:], bfront)):
    T = T.copy(); T[:, :4] -= T[:, 0].min()
    print(name, "span", T[:, 3].max() / 1e3, "us")
    lv = level[fr]
    for L in sorted(set(lv.tolist())):
        m = lv == L
        print(f"  level {L:2d} fronts {lvl_count[L]:5d} items {m.sum():6d} start {T[m,0].min()/1e3:8.1f} end {T[m,3].max()/1e3:8.1f} "
              f"busy {(T[m,3]-T[m,0]).sum()/1e3:8.1f} waited {T[m,5].sum()/1e3:7.1f} mean item {(T[m,3]-T[m,0]).mean()/1e3:6.2f} us")
if len(sys.argv) > 4:
    L = int(sys.argv[4])
    for name, T, fr in (("fwd", t[:nf_], ffront), ("bwd", t[nf_:], bfront)):
        T = T.copy(); T[:, :4] -= T[:, 0].min()
        base = (t[:nf_] if name == "fwd" else t[nf_:])[:, 0].min()
        for k in (4, 6, 7): T[:, k] = np.where(T[:, k] > 0, T[:, k] - base, -1)
        idx = np.nonzero(level[fr] == L)[0]
        idx = idx[np.argsort(T[idx, 0])][:40]
        print(name, "items of level", L, "(t0 t1 t2 t3 waited, us)")
        for i in idx:
            print(f"   item {i:6d} front {fr[i]:5d} {T[i,0]/1e3:8.2f} {T[i,1]/1e3:8.2f} {T[i,2]/1e3:8.2f} {T[i,3]/1e3:8.2f} w {T[i,5]/1e3:6.2f} detect {T[i,4]/1e3:8.2f} streamed {T[i,6]/1e3:8.2f} tri {T[i,7]/1e3:8.2f}")
if len(sys.argv) > 5:
    L = int(sys.argv[5])
    for name, T, fr in (("fwd", t[:nf_], ffront), ("bwd", t[nf_:], bfront)):
        m = level[fr] == L
        T = T[m].astype(float)
        ph = {"t0-t1 (pop..prologue)": T[:,1]-T[:,0], "t1-t6 (stream)": T[:,6]-T[:,1], "t6-t7 (tri)": T[:,7]-T[:,6],
              "t7-t2 (rest)": T[:,2]-T[:,7], "t2-t3 (publish)": T[:,3]-T[:,2]}
        print(name, "level", L, " ".join(f"{k}: {np.median(v)/1e3:.2f}" for k, v in ph.items()), "us (median)")
