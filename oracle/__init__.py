"""ORACLE — test infrastructure only (see oracle/rq_oracle.cpp header).

ctypes access to the CPU restatement (liboracle.so) and to the reference's own
sources built by oracle/Makefile (_ref/liboracle_ref.so). Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs may import this.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "liboracle_ref.so")

vp = C.c_void_p
i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def _bind(lib):
    def s(name, res, *args):
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = list(args)
    s("oracle_last_error", C.c_char_p)
    s("oracle_kind", C.c_int)
    s("oracle_symbolic", C.c_int, C.c_int64, i64p, i32p, i32p, C.c_int, C.c_int, i32p,
      C.POINTER(C.c_int32), i32p, i32p, i32p, C.POINTER(C.c_int64))
    s("oracle_factor_create", C.c_int, C.c_int64, i64p, i32p, f64p, i32p, C.c_int, C.c_int,
      C.POINTER(vp), C.POINTER(C.c_int64), C.POINTER(C.c_double))
    s("oracle_factor_solve", C.c_int, vp, f64p, f64p)
    s("oracle_factor_front", C.c_int, vp, C.c_int, vp, vp, vp)
    s("oracle_factor_destroy", None, vp)
    s("oracle_eig_create", C.c_int, C.c_int64, i64p, i32p, f64p, f64p, f64p, i32p, C.c_int,
      C.c_int, C.c_double, C.POINTER(vp))
    s("oracle_eig_factor_ms", C.c_double, vp)
    s("oracle_eig_apply", C.c_int, vp, f64p, f64p)
    s("oracle_eig_solve_quadratic", C.c_int, vp, C.c_int, C.c_int, C.c_double, C.c_uint64,
      C.c_int, C.c_int, f64p, f64p, vp, i32p, f64p)
    s("oracle_eig_solve_quadratic_block", C.c_int, vp, C.c_int, C.c_int, C.c_double, C.c_uint64,
      C.c_int, C.c_int, C.c_int, C.c_int, f64p, f64p, vp, i32p, f64p)
    s("oracle_eig_destroy", None, vp)
    s("oracle_gh_solve", C.c_int, C.c_int64, i64p, i32p, f64p, f64p, i32p, C.c_int, C.c_int, C.c_double,
      C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_int, f64p, f64p, i32p)
    s("oracle_eig_create2", C.c_int, vp, C.c_int64, i64p, i32p, f64p, f64p, f64p, i32p, C.c_int,
      C.c_int, C.c_double, C.c_int, C.POINTER(vp))
    s("oracle_eig_varsigma", C.c_double, vp)
    s("oracle_scale_pencil", C.c_int, C.c_int64, i64p, i32p, f64p, f64p, f64p, C.POINTER(C.c_double))
    s("oracle_symbolic_fronts", C.c_int, vp, C.POINTER(C.c_int32), vp, vp)
    s("oracle_eig_b_inner", C.c_int, vp, f64p, f64p, f64p)
    s("oracle_eig_arnoldi", C.c_int, vp, f64p, C.c_int, vp, vp)
    s("oracle_eig_ledger", None, vp, f64p)
    s("oracle_eig_ledger_reset", None, vp)
    s("oracle_eig_step_profile", C.c_int, vp, C.c_int, C.c_int, C.c_uint64, f64p)
    s("oracle_symbolic_create", C.c_int, C.c_int64, i64p, i32p, i32p, C.c_int, C.c_int, C.POINTER(vp))
    s("oracle_symbolic_destroy", None, vp)
    s("oracle_factor_numeric", C.c_int, vp, C.c_int64, i64p, i32p, f64p, C.POINTER(vp),
      C.POINTER(C.c_int64), C.POINTER(C.c_double))
    s("oracle_kern_spmv", None, C.c_int64, i64p, i32p, f64p, f64p, f64p)
    s("oracle_kern_dotc", None, f64p, f64p, C.c_int64, f64p)
    s("oracle_kern_elim", C.c_uint64, f64p, C.c_int64, f64p, f64p, C.c_int64, C.c_int64)
    return lib


_port = None
_ref = None


def port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_PATH):
            raise ImportError(f"{PORT_PATH} missing: run make -C oracle")
        _port = _bind(C.CDLL(PORT_PATH))
    return _port


def ref():
    """The reference-sources build, or None when it was never built here."""
    global _ref
    if _ref is None and os.path.exists(REF_PATH):
        lib = _bind(C.CDLL(REF_PATH))
        lib.ref_space.restype = C.c_int
        lib.ref_space.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int64), vp, vp,
                                  C.POINTER(C.c_int64)]
        lib.ref_kern_backend.restype = C.c_char_p
        lib.ref_kern_spmv.argtypes = [C.c_int64, i64p, i32p, f64p, f64p, f64p]
        lib.ref_kern_spmv.restype = None
        lib.ref_kern_dotc.argtypes = [f64p, f64p, C.c_int64, f64p]
        lib.ref_kern_dotc.restype = None
        lib.ref_kern_elim.argtypes = [f64p, C.c_int64, f64p, f64p, C.c_int64, C.c_int64]
        lib.ref_kern_elim.restype = C.c_uint64
        lib.ref_select_backend.argtypes = [C.c_char_p]
        lib.ref_select_backend.restype = C.c_int
        if hasattr(lib, "ref_mm_write"):  # Matrix Market through the reference's sparse.cpp
            lib.ref_mm_write.argtypes = [C.c_int64, i64p, i32p, f64p, vp, C.c_char_p]
            lib.ref_mm_write.restype = C.c_int
            lib.ref_mm_write_vector.argtypes = [C.c_int64, f64p, vp, C.c_char_p]
            lib.ref_mm_write_vector.restype = C.c_int
            lib.ref_mm_read.argtypes = [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), vp, vp, vp, vp]
            lib.ref_mm_read.restype = C.c_int
        _ref = lib
    return _ref


def lib_for(kind: str = "port"):
    if kind == "reference":
        r = ref()
        if r is None:
            raise ImportError("oracle/_ref/liboracle_ref.so not built")
        return r
    return port()


def _chk(lib, rc):
    if rc != 0:
        raise OracleError(rc, lib.oracle_last_error().decode())


def cplx(a) -> np.ndarray:
    """Interleave a real or complex array as (re, im) doubles."""
    a = np.asarray(a)
    out = np.zeros(2 * a.size)
    out[0::2] = a.real.ravel()
    if np.iscomplexobj(a):
        out[1::2] = a.imag.ravel()
    return out


def uncplx(a) -> np.ndarray:
    return a[0::2] + 1j * a[1::2]


def symbolic(pencil, leaf=64, kind="port"):
    lib = lib_for(kind)
    n = pencil.n
    perm = np.zeros(n, np.int32)
    nfr = C.c_int32()
    npiv = np.zeros(n + 1, np.int32)
    nf = np.zeros(n + 1, np.int32)
    parent = np.zeros(n + 1, np.int32)
    snnz = C.c_int64()
    _chk(lib, lib.oracle_symbolic(n, pencil.rowptr, pencil.col, np.ascontiguousarray(pencil.box.ravel(), np.int32),
                                  pencil.elems, leaf, perm, C.byref(nfr), npiv, nf, parent, C.byref(snnz)))
    k = nfr.value
    return {"perm": perm, "npiv": npiv[:k], "nf": nf[:k], "parent": parent[:k],
            "struct_nnz_l": snnz.value}


class Symbolic:
    """Oracle symbolic analysis (ND ordering + elimination-tree fronts) as a
    handle, reused by numeric factorizations (Factor(..., symbolic=S))."""

    def __init__(self, n, rowptr, col, box, elems, leaf=64, kind="port"):
        self.lib = lib_for(kind)
        self.n = n
        self.h = vp()
        _chk(self.lib, self.lib.oracle_symbolic_create(
            n, np.ascontiguousarray(rowptr, np.int64), np.ascontiguousarray(col, np.int32),
            np.ascontiguousarray(np.asarray(box).ravel(), np.int32), elems, leaf, C.byref(self.h)))

    def fronts(self):
        """(npiv, nf) per front, postorder."""
        k = C.c_int32()
        _chk(self.lib, self.lib.oracle_symbolic_fronts(self.h, C.byref(k), None, None))
        npiv, nf = np.zeros(k.value, np.int32), np.zeros(k.value, np.int32)
        _chk(self.lib, self.lib.oracle_symbolic_fronts(self.h, C.byref(k), npiv.ctypes.data_as(vp),
                                                       nf.ctypes.data_as(vp)))
        return npiv, nf

    def flops_lu(self):
        """F_LU = sum_f sum_{k<npiv} (nf-k-1) + 2 (nf-k-1)^2 (real flops)."""
        npiv, nf = self.fronts()
        tot = 0.0
        for p, n in zip(npiv.tolist(), nf.tolist()):
            r = np.arange(n - 1, n - 1 - p, -1, dtype=np.float64)
            tot += float(np.sum(r + 2 * r * r))
        return tot

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.oracle_symbolic_destroy(self.h)
            self.h = None


def scale_pencil(n, rowptr, col, K, C_, M, kind="port"):
    """scale_pencil: (varsigma, varsigma C, varsigma^2 M)."""
    lib = lib_for(kind)
    c, m = cplx(C_), cplx(M)
    vs = C.c_double()
    _chk(lib, lib.oracle_scale_pencil(n, np.ascontiguousarray(rowptr, np.int64), np.ascontiguousarray(col, np.int32),
                                      cplx(K), c, m, C.byref(vs)))
    return vs.value, uncplx(c), uncplx(m)


class Factor:
    """Oracle multifrontal LU (complex, reference elim_step inner loop)."""

    def __init__(self, n, rowptr, col, values, box=None, elems=None, leaf=64, kind="port", symbolic=None):
        self.lib = lib_for(kind)
        self.n = n
        self.h = vp()
        sw, macs = C.c_int64(), C.c_double()
        if symbolic is not None:
            _chk(self.lib, self.lib.oracle_factor_numeric(
                symbolic.h, n, np.ascontiguousarray(rowptr, np.int64), np.ascontiguousarray(col, np.int32),
                cplx(values), C.byref(self.h), C.byref(sw), C.byref(macs)))
        else:
            _chk(self.lib, self.lib.oracle_factor_create(
                n, np.ascontiguousarray(rowptr, np.int64), np.ascontiguousarray(col, np.int32),
                cplx(values), np.ascontiguousarray(np.asarray(box).ravel(), np.int32), elems, leaf,
                C.byref(self.h), C.byref(sw), C.byref(macs)))
        self.swaps, self.fa_macs = sw.value, macs.value

    def solve(self, b):
        x = np.zeros(2 * self.n)
        _chk(self.lib, self.lib.oracle_factor_solve(self.h, cplx(b), x))
        return uncplx(x)

    def front(self, f, nf, npiv):
        dense = np.zeros(2 * nf * nf)
        ipiv = np.zeros(max(npiv, 1), np.int32)
        rows = np.zeros(nf, np.int32)
        _chk(self.lib, self.lib.oracle_factor_front(self.h, f, dense.ctypes.data_as(vp),
                                                    ipiv.ctypes.data_as(vp), rows.ctypes.data_as(vp)))
        return uncplx(dense).reshape(nf, nf), ipiv[:npiv], rows

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.oracle_factor_destroy(self.h)
            self.h = None


class Eig:
    """Oracle quadratic eigensolver (complex Krylov-Schur, CGS2, guard)."""

    def __init__(self, pencil, sigma, leaf=64, kind="port", K=None, C_=None, M=None, scaling=False,
                 symbolic=None):
        self.lib = lib_for(kind)
        self.n = pencil.n
        self.h = vp()
        K = pencil.K if K is None else K
        C_ = pencil.C if C_ is None else C_
        M = pencil.M if M is None else M
        _chk(self.lib, self.lib.oracle_eig_create2(
            None if symbolic is None else symbolic.h, pencil.n, np.ascontiguousarray(pencil.rowptr, np.int64),
            np.ascontiguousarray(pencil.col, np.int32), cplx(K), cplx(C_), cplx(M),
            np.ascontiguousarray(np.asarray(pencil.box).ravel(), np.int32), pencil.elems, leaf, float(sigma),
            int(bool(scaling)), C.byref(self.h)))
        self.factor_ms = self.lib.oracle_eig_factor_ms(self.h)
        self.varsigma = self.lib.oracle_eig_varsigma(self.h)

    def apply(self, v):
        r = np.zeros(4 * self.n)
        _chk(self.lib, self.lib.oracle_eig_apply(self.h, cplx(v), r))
        return uncplx(r)

    LEDGER = ("fa", "fb", "mv", "vv", "residual_check", "restart")

    def ledger_counts(self):
        """Cumulative CostLedger counters of this operator: {cat: (ops, macs)}."""
        out = np.zeros(12)
        self.lib.oracle_eig_ledger(self.h, out)
        return {nm: (int(out[2 * i]), float(out[2 * i + 1])) for i, nm in enumerate(self.LEDGER)}

    def ledger_reset(self):
        self.lib.oracle_eig_ledger_reset(self.h)

    def b_inner(self, x, y):
        out = np.zeros(2)
        _chk(self.lib, self.lib.oracle_eig_b_inner(self.h, cplx(x), cplx(y), out))
        return out[0] + 1j * out[1]

    def arnoldi(self, v1, m):
        """(V (m+1) x 2n, H (m+1) x m) of arnoldi_run from v1."""
        n2 = 2 * self.n
        V = np.zeros(2 * (m + 1) * n2)
        H = np.zeros(2 * (m + 1) * m)
        _chk(self.lib, self.lib.oracle_eig_arnoldi(self.h, cplx(v1), m, V.ctypes.data_as(vp), H.ctypes.data_as(vp)))
        return uncplx(V).reshape(m + 1, n2), uncplx(H).reshape(m, m + 1).T

    def step_profile(self, j0, nsteps, seed=0):
        """ms in {spmv, solve, cgs2, other} over Arnoldi steps j0..j0+nsteps-1."""
        out = np.zeros(4)
        _chk(self.lib, self.lib.oracle_eig_step_profile(self.h, j0, nsteps, seed, out))
        return dict(zip(("spmv", "solve", "cgs2", "other"), out.tolist()))

    def solve_quadratic(self, nev, m=0, tol=1e-10, seed=0, max_restarts=100, guard=1,
                        vectors=False, block=1, block_min_steps=1):
        """block > 1: the block Krylov-Schur mode, the B200
        build's block algorithm operation for operation."""
        lam = np.zeros(2 * nev)
        res = np.zeros(nev)
        vec = np.zeros(2 * nev * self.n) if vectors else None
        st = np.zeros(4, np.int32)
        led = np.zeros(12)
        rc = self.lib.oracle_eig_solve_quadratic_block(self.h, nev, m, tol, seed, max_restarts, guard,
                                                       int(block), int(block_min_steps), lam, res,
                                                       None if vec is None else vec.ctypes.data_as(vp), st, led)
        self.stats = {"cycles": int(st[0]), "guard_passes": int(st[1]), "nconv": int(st[2]),
                      "ok": bool(st[3])}
        names = ["fa", "fb", "mv", "vv", "residual_check", "restart"]
        self.ledger = {nm: {"ops": int(led[2 * i]), "macs": float(led[2 * i + 1])}
                       for i, nm in enumerate(names)}
        _chk(self.lib, rc)
        out = uncplx(lam)
        if vectors:
            return out, res, uncplx(vec).reshape(nev, self.n)
        return out, res

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.oracle_eig_destroy(self.h)
            self.h = None


# --------------------------------------------------------------------------- assembly
# BASELINE.json configs by short name: (kind 0 curl / 1 div, p, ne, rIGA levels);
# restated here so the reference CPU arm never loads the product library.
CONFIGS = {
    "cfg1": (1, 2, 32, 0), "cfg2_iga": (1, 3, 64, 0), "cfg2_riga": (1, 3, 64, 3),
    "cfg3_iga": (0, 4, 128, 0), "cfg3_riga": (0, 4, 128, 3),
    "cfg4_iga": (1, 3, 512, 0), "cfg4_riga": (1, 3, 512, 5),
}
for _p in (2, 3, 4, 5):
    CONFIGS[f"cfg5_p{_p}_iga"] = (0, _p, 256, 0)
    CONFIGS[f"cfg5_p{_p}_riga"] = (0, _p, 256, 5)


class RefPencil:
    """BASELINE pencil assembled by oracle/ref_assembly.cpp on the reference's
    own spaces / splines / Piola code (an independent second route to the
    product's assembler). Same attribute names as the product's pencil."""

    def __init__(self, kind, degree, elems, levels=0, alpha=0.05, beta=0.01):
        lib = ref()
        if lib is None:
            raise ImportError("oracle/_ref/liboracle_ref.so not built")
        lib.ref_assemble.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.POINTER(vp)]
        lib.ref_assemble.restype = C.c_int
        lib.ref_assemble_last_error.restype = C.c_char_p
        lib.ref_assemble_dims.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        lib.ref_assemble_dims.restype = None
        lib.ref_assemble_copy.argtypes = [vp, i64p, i32p, f64p, f64p, f64p, i32p]
        lib.ref_assemble_copy.restype = None
        lib.ref_assemble_destroy.argtypes = [vp]
        lib.ref_assemble_destroy.restype = None
        h = vp()
        rc = lib.ref_assemble(kind, degree, elems, levels, alpha, beta, C.byref(h))
        if rc != 0:
            raise OracleError(rc, lib.ref_assemble_last_error().decode())
        nf, n, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        lib.ref_assemble_dims(h, C.byref(nf), C.byref(n), C.byref(nnz))
        self.n_full, self.n, self.nnz = nf.value, n.value, nnz.value
        self.rowptr = np.zeros(self.n + 1, np.int64)
        self.col = np.zeros(self.nnz, np.int32)
        self.K, self.C, self.M = (np.zeros(self.nnz) for _ in range(3))
        self.box = np.zeros((self.n, 4), np.int32)
        lib.ref_assemble_copy(h, self.rowptr, self.col, self.K, self.C, self.M, self.box)
        lib.ref_assemble_destroy(h)
        self.elems, self.degree, self.kind, self.levels = elems, degree, kind, levels

    def q_values(self, sigma):
        return self.K + sigma * self.C + sigma * sigma * self.M


def ref_config(name):
    return RefPencil(*CONFIGS[name])


def solve_generalized_hermitian(rowptr, col, A, B, box, elems, s, nev, m=0, tol=1e-10, seed=0, max_restarts=100,
                                leaf=64, kind="port"):
    """Oracle restatement of solve_generalized_hermitian:
    complex multifrontal LU of A - s B, Lanczos with full reorthogonalisation,
    thick restarts. Returns (lam, res) nearest the shift first."""
    lib = lib_for(kind)
    n = len(rowptr) - 1
    lam, res, st = np.zeros(nev), np.zeros(nev), np.zeros(2, np.int32)
    _chk(lib, lib.oracle_gh_solve(n, np.ascontiguousarray(rowptr, np.int64), np.ascontiguousarray(col, np.int32),
                                  np.ascontiguousarray(A, np.float64), np.ascontiguousarray(B, np.float64),
                                  np.ascontiguousarray(np.asarray(box).ravel(), np.int32), int(elems), int(leaf),
                                  float(s), int(nev), int(m), float(tol), int(seed), int(max_restarts), lam, res, st))
    return lam, res

