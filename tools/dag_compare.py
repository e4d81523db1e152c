import sys, numpy as np
a = np.load("gpurun_out/dbg_dag.npy", allow_pickle=True).item()
b = np.load("gpurun_out/dbg_level.npy", allow_pickle=True).item()
print("dag", a["info"], "level", b["info"])
for i, (fa, fb) in enumerate(zip(a["fronts"], b["fronts"])):
    nf, np_, lev, par, Fa, pa = fa
    Fb, pb = fb[4], fb[5]
    d = np.abs(Fa - Fb)
    m = d.max() / max(np.abs(Fb).max(), 1e-300)
    if m > 1e-9 or not np.array_equal(pa, pb):
        r, c = np.unravel_index(np.argmax(d), d.shape)
        bad = np.argwhere(d > 1e-9 * np.abs(Fb).max())
        print(f"front {i} nf={nf} npiv={np_} lev={lev} parent={par} relerr={m:.2e} at ({r},{c}); ipiv_eq={np.array_equal(pa,pb)}; nbad={len(bad)} rows[{bad[:,0].min()}..{bad[:,0].max()}] cols[{bad[:,1].min()}..{bad[:,1].max()}]")
        if i > 40: break
