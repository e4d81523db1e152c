"""e2e refactor from pinned host values (development aid): wall ms per refactor,
streamed upload (default) against RQB_STREAM_UPLOAD=0, and the factors compared.
python tools/e2e_refactor.py cfg4_riga [reps]"""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_2112_14064_b200 as rq
cfg = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
P = rq.baseline_config(cfg)
o = rq.nested_dissection_order(P)
Q = P.q_values(-0.5)
pin = torch.empty(P.nnz, dtype=torch.float64, pin_memory=True)
pin.copy_(torch.from_numpy(Q))
Qh = pin.numpy()
fac = rq.lu_factorize((P.rowptr, P.col, Qh), o)
b = np.random.default_rng(0).uniform(-1, 1, P.n)
for _ in range(3):
    fac.refactor(Qh)
t0 = time.perf_counter()
for _ in range(reps):
    fac.refactor(Qh)
ms = (time.perf_counter() - t0) * 1e3 / reps
x = fac.solve(b)
import scipy.sparse as sp
A = sp.csr_matrix((Q, P.col, P.rowptr), shape=(P.n, P.n))
r = A @ x - b
berr = np.abs(r).max() / (abs(A).dot(np.abs(x)) + np.abs(b)).max()
print(f"{cfg}: e2e refactor {ms:.3f} ms ({o.stats['flops_lu'] / ms / 1e6:.1f} GF/s), device window {fac.info()['factor_ms']:.3f} ms, "
      f"solve backward error {berr:.2e}, x checksum {float(np.sum(x)):.15e}")
