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

    def b_inner(self, x: np.ndarray, y: np.ndarray) -> float:
        out = C.c_double()
        check(_lib.lib.rq_operator_b_inner(self._h, np.ascontiguousarray(x, np.float64),
                                           np.ascontiguousarray(y, np.float64), C.byref(out)))
        return out.value

    def spmv(self, which: str, x: np.ndarray) -> np.ndarray:
        w = {"K": 0, "C": 1, "M": 2, "Q": 3}[which]
        y = np.zeros(self.n)
        check(_lib.lib.rq_operator_spmv(self._h, w, np.ascontiguousarray(x, np.float64), y))
        return y

    def arnoldi(self, v1: np.ndarray, m: int):
        V = np.zeros((m + 1, 2 * self.n))
        H = np.zeros(m * (m + 1))
        check(_lib.lib.rq_operator_arnoldi(self._h, np.ascontiguousarray(v1, np.float64), int(m),
                                           _lib.ptr(V), _lib.ptr(H)))
        return V, H.reshape(m, m + 1).T

    def factor_info(self) -> dict:
        from ._lib import FactorInfo
        fi = FactorInfo()
        check(_lib.lib.rq_factor_get_info(_lib.lib.rq_operator_factor(self._h), C.byref(fi)))
        return {k: getattr(fi, k) for k, _ in FactorInfo._fields_}

    def solve_quadratic(self, nev: int, m: int = 0, eps: float = 1e-10, seed: int = 0,
                        max_restarts: int = 100, guard: bool = True, vectors: bool = False,
                        raise_partial: bool = True, profile: bool = False):
        n = self.n
        lr, li, rs = np.zeros(nev), np.zeros(nev), np.ones(nev)
        vr = np.zeros(n * nev) if vectors else None
        vi = np.zeros(n * nev) if vectors else None
        opts = EigsOpts(int(nev), int(m), float(eps), int(seed), int(max_restarts), 1 if guard else 0,
                        1 if profile else 0)
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
        if h is not None and h.value:
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


def solve_quadratic(pencil, s: float, nev: int, m: int = 0, eps: float = 1e-10, seed: int = 0,
                    ordering: Ordering | None = None, scaling: bool = False, **kw):
    """SPEC.md:462 solve_quadratic(pencil, s, nev, m, eps) -> list of EigenPair."""
    op = build_operator(pencil, s, ordering, scaling)
    return op.solve_quadratic(nev, m, eps, seed, **kw), op
