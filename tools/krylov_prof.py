"""Krylov vector-kernel timing per config (development aid): fused C/M SpMV,
M SpMV, CGS GEMV-T / GEMV-N at several basis sizes, with an L2 scrub per call."""
import ctypes as C
import sys
sys.path.insert(0, ".")
import paper_2112_14064_b200 as rq
from paper_2112_14064_b200 import _lib
for cfg in sys.argv[1:]:
    P = rq.baseline_config(cfg)
    op = rq.build_operator(P, -0.5)
    n, nnz = P.n, P.nnz
    def t(what, iters, param=0):
        ms = C.c_double()
        _lib.check(_lib.lib.rq_operator_time(op._h, what | 0x100, iters, param, C.byref(ms)))
        return ms.value
    sp = t(2, 20); sm = t(6, 20)
    b_sp = 20 * nnz + 8 * (n + 1) + 24 * n
    b_sm = 12 * nnz + 8 * (n + 1) + 16 * n
    print(f"{cfg}: n {n} nnz {nnz}  spmv_fused {sp*1e3:.1f} us {b_sp/sp/1e6:.0f} GB/s  spmv_M {sm*1e3:.1f} us {b_sm/sm/1e6:.0f} GB/s")
    for k in (10, 41, 101, 201):
        gt, gn = t(3, 10, k), t(4, 10, k)
        b = 8 * 2 * n * k
        print(f"   k={k:3d} gemv_t {gt*1e3:8.1f} us {b/gt/1e6:6.0f} GB/s   gemv_n {gn*1e3:8.1f} us {(b + 16*2*n)/gn/1e6:6.0f} GB/s")
    for k in (41, 201):
        if k > 2 * 41 and n < 100000: continue
        gm = t(7, 5, k); rs = t(8, 3, k)
        print(f"   restart dgemm 2n x {k} x {k}: {gm*1e3:8.1f} us {2*2*n*k*k/gm/1e9:6.1f} TFLOP/s;  residual batch of {k}: {rs*1e3:8.1f} us ({rs*1e3/k:.1f} us/cand)")
