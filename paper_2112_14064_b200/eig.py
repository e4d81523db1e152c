"""eig: the quadratic shift-invert Krylov-Schur eigensolver (SPEC.md:380-511,
PAPER.md Alg. 2 :555-589) over the B200 C-ABI.

build_operator factors Q(s) = K + sC + s^2 M on the GPU (N_fa = 1);
apply_operator / b_inner / arnoldi_run expose the device kernels for parity
tests; solve_quadratic runs the whole device-resident eigensolve.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import EigsInfo, EigsOpts, OperatorOpts, RqError, check
from .sparsela import Ordering, nested_dissection_order


LEDGER_CATEGORIES = ("fa", "fb", "mv", "vv", "residual_check", "restart")


@dataclass
class EigenPair:
    lam: complex
    residual: float
    u: np.ndarray | None = None


class ShiftInvertOperator:
    """S = L(s)^{-1} B of the linearised pencil, device resident."""

    def __init__(self, pencil, s: float, ordering: Ordering | None = None, scaling: bool = False):
        if isinstance(s, complex):
            if s.imag != 0:
                raise RqError(2, "the B200 path takes real shifts only")
            s = s.real
        resident = getattr(pencil, "device_resident", False)
        if not resident:
            for arr in (pencil.K, pencil.C, pencil.M):
                if np.iscomplexobj(arr) and np.any(arr.imag != 0):
                    raise RqError(2, "the B200 path takes real pencils only")
        self.pencil = pencil
        self.s = float(s)
        self.ordering = ordering if ordering is not None else nested_dissection_order(pencil)
        self.n = pencil.n
        opts = OperatorOpts(float(s), 1 if scaling else 0)
        self._h = C.c_void_p()
        if resident:  # device-assembled K, C, M used in place
            check(_lib.lib.rq_operator_create_pencil(pencil.handle, self.ordering.handle, C.byref(opts),
                                                     C.byref(self._h)))
        else:
            check(_lib.lib.rq_operator_create(
                pencil.n, np.ascontiguousarray(pencil.rowptr, np.int64),
                np.ascontiguousarray(pencil.col, np.int32), np.ascontiguousarray(pencil.K, np.float64),
                np.ascontiguousarray(pencil.C, np.float64), np.ascontiguousarray(pencil.M, np.float64),
                self.ordering.handle, C.byref(opts), C.byref(self._h)))
        self.varsigma = _lib.lib.rq_operator_varsigma(self._h)
        self.last_info: dict = {}
        self.ledger: dict = {}

    # --- SPEC operations ---------------------------------------------------
    def apply(self, v: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(v, np.float64)
        if v.size != 2 * self.n:
            raise RqError(7, "apply_operator dimension mismatch")
        r = np.zeros_like(v)
        check(_lib.lib.rq_operator_apply(self._h, v, r))
        return r

    def _vec(self, x, size, what):
        x = np.ascontiguousarray(x, np.float64)
        if x.ndim != 1 or x.size != size:
            raise RqError(7, f"{what} dimension mismatch: {x.size} entries, expected {size}")
        return x

    def b_inner(self, x: np.ndarray, y: np.ndarray) -> float:
        x = self._vec(x, 2 * self.n, "b_inner")
        y = self._vec(y, 2 * self.n, "b_inner")
        out = C.c_double()
        check(_lib.lib.rq_operator_b_inner(self._h, x, y, C.byref(out)))
        return out.value

    def spmv(self, which: str, x: np.ndarray) -> np.ndarray:
        w = {"K": 0, "C": 1, "M": 2, "Q": 3}[which]
        x = self._vec(x, self.n, "spmv")
        y = np.zeros(self.n)
        check(_lib.lib.rq_operator_spmv(self._h, w, x, y))
        return y

    def arnoldi(self, v1: np.ndarray, m: int):
        v1 = self._vec(v1, 2 * self.n, "arnoldi_run")
        if not 1 <= m < 2 * self.n:
            raise RqError(2, "arnoldi_run: m must be in [1, 2n)")
        V = np.zeros((m + 1, 2 * self.n))
        H = np.zeros(m * (m + 1))
        check(_lib.lib.rq_operator_arnoldi(self._h, v1, int(m), _lib.ptr(V), _lib.ptr(H)))
        return V, H.reshape(m, m + 1).T

    def ritz_extract(self, H: np.ndarray):
        """SPEC.md:444 ritz_extract of an (m+1) x m Hessenberg of this operator."""
        return ritz_extract(H, self.s, self.varsigma)

    def krylov_schur_restart(self, V: np.ndarray, H: np.ndarray, keep: int):
        """SPEC.md:453 krylov_schur_restart: (V[:p+1], H[:p+1, :p], p)."""
        V = np.array(V, dtype=np.float64, order="C", copy=True)
        H = np.asarray(H, np.float64)
        m = H.shape[1]
        if H.shape != (m + 1, m) or V.shape != (m + 1, 2 * self.n):
            raise RqError(7, "krylov_schur_restart: V must be (m+1) x 2n and H (m+1) x m")
        Hc = np.array(H.T, dtype=np.float64, order="C")  # column-major (m+1) x m
        p = C.c_int()
        check(_lib.lib.rq_operator_krylov_schur_restart(self._h, m, int(keep), V.reshape(-1), Hc.reshape(-1),
                                                        C.byref(p)))
        p = p.value
        Hn = Hc.reshape(m, m + 1).T
        return V[:p + 1], Hn[:p + 1, :p], p

    def ledger_counts(self) -> dict:
        """Cumulative CostLedger of this operator: {category: (ops, macs)}."""
        out = np.zeros(12)
        check(_lib.lib.rq_operator_ledger(self._h, out))
        return {nm: (int(out[2 * i]), float(out[2 * i + 1])) for i, nm in enumerate(LEDGER_CATEGORIES)}

    def ledger_json(self) -> dict:
        buf = C.create_string_buffer(4096)
        check(_lib.lib.rq_operator_ledger_json(self._h, buf, 4096))
        return json.loads(buf.value.decode())

    def release_workspace(self) -> None:
        """Free the Krylov workspace kept across solve_quadratic calls."""
        check(_lib.lib.rq_operator_release_workspace(self._h))

    def ledger_reset(self) -> None:
        check(_lib.lib.rq_operator_ledger_reset(self._h))

    def factor_info(self) -> dict:
        from ._lib import FactorInfo
        fi = FactorInfo()
        check(_lib.lib.rq_factor_get_info(_lib.lib.rq_operator_factor(self._h), C.byref(fi)))
        return {k: getattr(fi, k) for k, _ in FactorInfo._fields_}

    def solve_quadratic(self, nev: int, m: int = 0, eps: float = 1e-10, seed: int = 0,
                        max_restarts: int = 100, guard: bool = True, vectors: bool = False,
                        raise_partial: bool = True, profile: bool = False, block: int = 1):
        """SPEC.md:462 solve_quadratic. block > 1 selects the block Krylov-Schur
        (block size 2..8: multi-RHS sweeps, block CGS2)."""
        n = self.n
        lr, li, rs = np.zeros(nev), np.zeros(nev), np.ones(nev)
        vr = np.zeros(n * nev) if vectors else None
        vi = np.zeros(n * nev) if vectors else None
        opts = EigsOpts(int(nev), int(m), float(eps), int(seed), int(max_restarts), 1 if guard else 0,
                        1 if profile else 0, int(block))
        info = EigsInfo()
        rc = _lib.lib.rq_eigs_run(self._h, C.byref(opts), _lib.ptr(lr), _lib.ptr(li), _lib.ptr(rs),
                                  _lib.ptr(vr), _lib.ptr(vi), C.byref(info))
        self.last_info = {k: getattr(info, k) for k, _ in EigsInfo._fields_}
        buf = C.create_string_buffer(4096)
        if _lib.lib.rq_eigs_ledger_json(self._h, buf, 4096) == 0:
            self.ledger = json.loads(buf.value.decode())
        if rc != 0 and (rc != 4 or raise_partial):
            check(rc)
        pairs = []
        for i in range(nev):
            u = None
            if vectors:
                u = vr[i * n:(i + 1) * n] + 1j * vi[i * n:(i + 1) * n]
            pairs.append(EigenPair(complex(lr[i], li[i]), float(rs[i]), u))
        return pairs

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None and _lib.lib is not None:  # (interpreter shutdown)
            _lib.lib.rq_operator_destroy(h)
            self._h = None


def build_operator(pencil, s: float, ordering: Ordering | None = None,
                   scaling: bool = False) -> ShiftInvertOperator:
    """SPEC.md:408 build_operator(pencil, s, ordering, counter)."""
    return ShiftInvertOperator(pencil, s, ordering, scaling)


def apply_operator(op: ShiftInvertOperator, v: np.ndarray) -> np.ndarray:
    """SPEC.md:417 r_u = -Q(s)^{-1}(s M v_u + C v_u + M v_l), r_l = s r_u + v_u."""
    return op.apply(v)


def b_inner(op: ShiftInvertOperator, x: np.ndarray, y: np.ndarray) -> float:
    """SPEC.md:426 x_u^T y_u + x_l^T M y_l (real build)."""
    return op.b_inner(x, y)


def arnoldi_run(op: ShiftInvertOperator, v1: np.ndarray, m: int):
    """SPEC.md:435 m-step B-orthogonal Arnoldi with CGS2: (V (m+1) x 2N, H (m+1) x m)."""
    return op.arnoldi(v1, m)


def scale_pencil(pencil):
    """SPEC.md:399 scale_pencil(pencil) -> (varsigma, C scaled, M scaled):
    varsigma = sqrt(maxabs K / maxabs M), scaled pencil (K, varsigma C,
    varsigma^2 M). Zero M raises RqError (domain)."""
    K = np.ascontiguousarray(pencil.K, np.float64)
    Cv = np.ascontiguousarray(pencil.C, np.float64)
    M = np.ascontiguousarray(pencil.M, np.float64)
    if not K.size == Cv.size == M.size:
        raise RqError(7, "scale_pencil: K, C, M must share one pattern")
    vs = C.c_double()
    Cs, Ms = np.empty_like(Cv), np.empty_like(M)
    check(_lib.lib.rq_scale_pencil(K.size, K, Cv, M, C.byref(vs), _lib.ptr(Cs), _lib.ptr(Ms)))
    return vs.value, Cs, Ms


def ritz_extract(H: np.ndarray, sigma: float, varsigma: float = 1.0) -> dict:
    """SPEC.md:444 ritz_extract: Ritz data of an (m+1) x m Hessenberg H in
    wanted order (nearest the shift first): theta, lambda = sigma + varsigma /
    theta, residual estimate |beta e_m^H y| and the unit Ritz vectors y (columns)."""
    H = np.asarray(H, np.float64)
    m = H.shape[1]
    if H.shape != (m + 1, m):
        raise RqError(7, "ritz_extract: H must be (m+1) x m")
    Hc = np.ascontiguousarray(H.T).reshape(-1)  # column-major
    th, lam, est, Y = np.zeros(2 * m), np.zeros(2 * m), np.zeros(m), np.zeros(2 * m * m)
    check(_lib.lib.rq_ritz_extract(Hc, m, float(sigma), float(varsigma), _lib.ptr(th), _lib.ptr(lam),
                                   _lib.ptr(est), _lib.ptr(Y)))
    Yc = (Y[0::2] + 1j * Y[1::2]).reshape(m, m).T
    return {"theta": th[0::2] + 1j * th[1::2], "lambda": lam[0::2] + 1j * lam[1::2], "est": est, "y": Yc}


def krylov_schur_restart(op: ShiftInvertOperator, V: np.ndarray, H: np.ndarray, keep: int):
    """SPEC.md:453 krylov_schur_restart(state, keep) -> (V_p+1, H_(p+1) x p, p)."""
    return op.krylov_schur_restart(V, H, keep)


def solve_quadratic(pencil, s: float, nev: int, m: int = 0, eps: float = 1e-10, seed: int = 0,
                    ordering: Ordering | None = None, scaling: bool = False, **kw):
    """SPEC.md:462 solve_quadratic(pencil, s, nev, m, eps) -> list of EigenPair."""
    op = build_operator(pencil, s, ordering, scaling)
    return op.solve_quadratic(nev, m, eps, seed, **kw), op


class GeneralizedHermitianSolver:
    """solve_generalized_hermitian on the device: A u = lambda B u,
    A symmetric, B symmetric positive definite on one CSR pattern, real shift s.
    A - s B is factored once (the multifrontal LU); shift-invert Lanczos with
    thick restarts runs on the device."""

    def __init__(self, rowptr, col, A, B, s: float, ordering: Ordering):
        from ._lib import GhInfo  # noqa: F401
        self.n = int(ordering.n)
        self.rowptr = np.ascontiguousarray(rowptr, np.int64)
        self.col = np.ascontiguousarray(col, np.int32)
        A = np.asarray(A)
        B = np.asarray(B)
        for X in (A, B):
            if np.iscomplexobj(X) and np.any(X.imag != 0):
                raise RqError(2, "the B200 path solves real symmetric problems only")
        A, B = np.ascontiguousarray(np.real(A), np.float64), np.ascontiguousarray(np.real(B), np.float64)
        nnz = int(self.rowptr[-1]) if self.rowptr.size else 0
        if self.rowptr.size != self.n + 1 or A.size != nnz or B.size != nnz or self.col.size != nnz:
            raise RqError(7, "solve_generalized_hermitian dimension mismatch")
        if not np.isfinite(s) or np.iscomplexobj(s):
            raise RqError(2, "the shift must be real")
        self.shift = float(s)
        self.ordering = ordering
        self._h = C.c_void_p()
        check(_lib.lib.rq_gh_create(self.n, self.rowptr, self.col, A, B, ordering.handle, self.shift,
                                    C.byref(self._h)))

    def solve(self, nev: int, m: int = 0, eps: float = 1e-10, seed: int = 0, max_restarts: int = 100,
              vectors: bool = False):
        from ._lib import GhInfo, GhOpts
        lam, res = np.zeros(nev), np.ones(nev)
        vec = np.zeros(self.n * nev) if vectors else None
        info = GhInfo()
        opts = GhOpts(int(nev), int(m), float(eps), int(seed), int(max_restarts))
        rc = _lib.lib.rq_gh_run(self._h, C.byref(opts), lam, res, _lib.ptr(vec), C.byref(info))
        self.last_info = {k: getattr(info, k) for k, _ in GhInfo._fields_}
        check(rc)
        return [EigenPair(complex(lam[i], 0.0), float(res[i]),
                          vec[i * self.n:(i + 1) * self.n].copy() if vectors else None) for i in range(nev)]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None and _lib.lib is not None:  # (interpreter shutdown)
            _lib.lib.rq_gh_destroy(h)
            self._h = None


def solve_generalized_hermitian(A, B, s: float, nev: int, m: int = 0, eps: float = 1e-10,
                                ordering: Ordering | None = None, seed: int = 0, max_restarts: int = 100,
                                vectors: bool = False, pencil=None):
    """SPEC.md:471 solve_generalized_hermitian(A, B, s_real, nev, m, eps, counter): A, B are
    (rowptr, col, values) on one pattern (or value arrays with `pencil` giving the pattern
    and the support boxes of the nested-dissection ordering)."""
    if pencil is not None:
        rowptr, col = pencil.rowptr, pencil.col
        Av, Bv = A, B
        if ordering is None:
            ordering = Ordering(pencil.n, pencil.box, pencil.elems)
    else:
        rowptr, col, Av = A
        _, _, Bv = B
    if ordering is None:
        raise RqError(2, "an Ordering (or a pencil) is required")
    solver = GeneralizedHermitianSolver(rowptr, col, Av, Bv, s, ordering)
    pairs = solver.solve(nev, m=m, eps=eps, seed=seed, max_restarts=max_restarts, vectors=vectors)
    solve_generalized_hermitian.last_info = solver.last_info
    return pairs



def solve_quadratic_complex(pencil, s: complex, nev: int, m: int = 0, eps: float = 1e-10, seed: int = 0,
                            max_restarts: int = 100, vectors: bool = False, K=None, C=None, M=None):
    """solve_quadratic for complex pencils and complex shifts (SURVEY.md
    §8 f4): K, C, M (default: the pencil's; any may be complex, e.g. the conductive
    EM damping C = -i sigma M_sigma) on the pencil's pattern, complex shift s. Q(s)
    is factored on the GPU as its real-equivalent 2n system; complex Krylov-Schur
    on the device. Returns EigenPair list (lam complex, residual, u complex)."""
    n = int(pencil.n)
    K = pencil.K if K is None else K
    C = pencil.C if C is None else C
    M = pencil.M if M is None else M

    def inter(a):
        a = np.asarray(a, np.complex128)
        return np.ascontiguousarray(np.stack([a.real, a.imag], 1).reshape(-1))
    Kc, Cc, Mc = inter(K), inter(C), inter(M)
    nnz = int(pencil.rowptr[-1])
    if Kc.size != 2 * nnz or Cc.size != 2 * nnz or Mc.size != 2 * nnz:
        raise RqError(7, "K, C, M must live on the pencil's pattern")
    o2 = Ordering(2 * n, np.repeat(np.asarray(pencil.box).reshape(-1, 4), 2, axis=0), pencil.elems)
    import ctypes  # (C is the damping matrix in this function)
    hh = ctypes.c_void_p()
    s = complex(s)
    check(_lib.lib.rq_zeig_create(o2.handle, n, np.ascontiguousarray(pencil.rowptr, np.int64),
                                  np.ascontiguousarray(pencil.col, np.int32), Kc, Cc, Mc, s.real, s.imag,
                                  ctypes.byref(hh)))
    try:
        lam = np.zeros(2 * nev)
        res = np.ones(nev)
        vec = np.zeros(2 * n * nev) if vectors else None
        st = np.zeros(2, np.int32)
        rc = _lib.lib.rq_zeig_run(hh, int(nev), int(m), float(eps), int(seed), int(max_restarts), lam, res,
                                  _lib.ptr(vec), st)
        solve_quadratic_complex.last_info = {"cycles": int(st[0]), "nconv": int(st[1])}
        check(rc)
    finally:
        _lib.lib.rq_zeig_destroy(hh)
    out = []
    for i in range(nev):
        u = None
        if vectors:
            u = vec[2 * n * i:2 * n * (i + 1)].view(np.complex128).copy()
        out.append(EigenPair(complex(lam[2 * i], lam[2 * i + 1]), float(res[i]), u))
    return out
