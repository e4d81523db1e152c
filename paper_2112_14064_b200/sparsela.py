"""sparsela: nested_dissection_order / lu_factorize / solve_factored
 over the B200 C-ABI.

Names, argument meaning and error behaviour follow SPEC's sparsela module:
errors raise RqError with the rq::errc category (singular -> code 8,
dimension mismatch -> 7, non-real input -> 2 config: the GPU path is real FP64
only).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import FactorInfo, RqError, SymbolicStats, check


class Ordering:
    """Geometric nested-dissection ordering + multifrontal front structure."""

    def __init__(self, n: int, box: np.ndarray, elems: int, leaf: int = 64):
        box = np.ascontiguousarray(box, dtype=np.int32).reshape(-1)
        if box.size != 4 * n:
            raise RqError(7, "support boxes must be n x 4")
        self._h = C.c_void_p()
        check(_lib.lib.rq_nd_order(int(n), box, int(elems), int(leaf), C.byref(self._h)))
        self.n, self.elems, self.leaf = int(n), int(elems), int(leaf)
        self.box = box.reshape(-1, 4)
        st = SymbolicStats()
        check(_lib.lib.rq_symbolic_stats_get(self._h, C.byref(st)))
        self.stats = {k: getattr(st, k) for k, _ in SymbolicStats._fields_}
        self.perm = np.zeros(n, np.int32)
        check(_lib.lib.rq_symbolic_perm(self._h, self.perm))
        nf = int(st.nfronts)
        self.parent = np.zeros(nf, np.int32)
        self.npiv = np.zeros(nf, np.int32)
        self.nf = np.zeros(nf, np.int32)
        self.start = np.zeros(nf, np.int32)
        self.level = np.zeros(nf, np.int32)
        check(_lib.lib.rq_symbolic_fronts(self._h, self.parent, self.npiv, self.nf, self.start,
                                          self.level))
        self.method = "geometric-nested-dissection"

    def front_rows(self, f: int) -> np.ndarray:
        out = np.zeros(int(self.nf[f]), np.int32)
        check(_lib.lib.rq_symbolic_front_rows(self._h, int(f), out))
        return out

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None and _lib.lib is not None:  # (interpreter shutdown)
            _lib.lib.rq_symbolic_destroy(h)
            self._h = None


def nested_dissection_order(pencil, leaf: int = 64) -> Ordering:
    """SPEC.md:302 nested_dissection_order(space) -> Ordering."""
    return Ordering(pencil.n, pencil.box, pencil.elems, leaf)


class Factorization:
    """Device-resident multifrontal LU of A (immutable; shareable read-only).
    A complex A (any nonzero imaginary part, e.g. Q(s) at a complex shift) is
    factored as its real-equivalent 2n system (rq_factor_create_complex): the
    2n unknowns (Re x_k, Im x_k) get their own nested-dissection ordering over
    the support boxes repeated per pair; solves take and return complex vectors."""

    def __init__(self, ordering: Ordering, rowptr, col, values):
        values = np.asarray(values)
        self.is_complex = bool(np.iscomplexobj(values) and np.any(values.imag != 0))
        if np.iscomplexobj(values) and not self.is_complex:
            values = values.real
        self.ordering = ordering
        self.n = ordering.n
        self.rowptr = np.ascontiguousarray(rowptr, np.int64)
        self.col = np.ascontiguousarray(col, np.int32)
        if self.rowptr.size != self.n + 1:
            raise RqError(7, "rowptr size does not match the ordering")
        self._h = C.c_void_p()
        if self.is_complex:
            self.ordering2 = Ordering(2 * self.n, np.repeat(ordering.box, 2, axis=0), ordering.elems,
                                      ordering.leaf)
            check(_lib.lib.rq_factor_create_complex(self.ordering2.handle, self.n, self.rowptr, self.col,
                                                    np.ascontiguousarray(values.real, np.float64),
                                                    _lib.ptr(np.ascontiguousarray(values.imag, np.float64)),
                                                    C.byref(self._h)))
            return
        check(_lib.lib.rq_factor_create(ordering.handle, self.n, self.rowptr, self.col,
                                        np.ascontiguousarray(values, np.float64),
                                        C.byref(self._h)))

    def info(self) -> dict:
        fi = FactorInfo()
        check(_lib.lib.rq_factor_get_info(self._h, C.byref(fi)))
        return {k: getattr(fi, k) for k, _ in FactorInfo._fields_}

    def refactor(self, values) -> None:
        check(_lib.lib.rq_factor_refactor(self._h, np.ascontiguousarray(values, np.float64)))

    def solve(self, b: np.ndarray, block: int | None = None) -> np.ndarray:
        """x = A^{-1} b; b of shape (n,) or (n, nrhs). Several right-hand sides
        pass through the multi-RHS sweeps, `block` (1..8, default 8) vectors per
        pass over the factors; block=1 forces the single-vector sweeps."""
        if self.is_complex:
            bc = np.asarray(b, dtype=np.complex128)
            if bc.shape[0] != self.n:
                raise RqError(7, "solve_factored dimension mismatch")
            bb = np.ascontiguousarray(bc.reshape(self.n, -1).T)  # nrhs x n complex = interleaved {re, im}
            x = np.zeros_like(bb)
            check(_lib.lib.rq_factor_solve_complex(self._h, bb.view(np.float64).reshape(-1),
                                                   x.view(np.float64).reshape(-1), bb.shape[0]))
            return x.T.reshape(bc.shape)
        if np.iscomplexobj(b):  # real factorization, complex right-hand side: two real solves
            return self.solve(np.real(b), block) + 1j * self.solve(np.imag(b), block)
        b = np.asarray(b, dtype=np.float64)
        if b.shape[0] != self.n:
            raise RqError(7, "solve_factored dimension mismatch")
        bb = np.ascontiguousarray(b.reshape(self.n, -1).T)
        x = np.zeros_like(bb)
        if block is None:
            block = 8 if bb.shape[0] > 1 else 1
        check(_lib.lib.rq_factor_solve_ex(self._h, bb, x, bb.shape[0], int(block)))
        return x.T.reshape(b.shape)

    def front(self, f: int):
        """(dense ld x nf column-major block, ipiv, ld) of front f after factorization."""
        nf = int(self.ordering.nf[f])
        ld = C.c_int64()
        check(_lib.lib.rq_factor_front_export(self._h, int(f), None, None, C.byref(ld)))
        dense = np.zeros(ld.value * nf)
        ipiv = np.zeros(max(1, int(self.ordering.npiv[f])), np.int32)
        check(_lib.lib.rq_factor_front_export(self._h, int(f), _lib.ptr(dense), _lib.ptr(ipiv),
                                              C.byref(ld)))
        return dense.reshape(nf, ld.value).T, ipiv[: int(self.ordering.npiv[f])], ld.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None and _lib.lib is not None:  # (interpreter shutdown)
            _lib.lib.rq_factor_destroy(h)
            self._h = None


def lu_factorize(A, ordering: Ordering) -> Factorization:
    """SPEC.md:311 lu_factorize(A, ord) -> Factorization. A: scipy CSR or (rowptr, col, val)."""
    if hasattr(A, "indptr"):
        A = A.tocsr()
        A.sort_indices()
        return Factorization(ordering, A.indptr, A.indices, A.data)
    rowptr, col, val = A
    return Factorization(ordering, rowptr, col, val)


def solve_factored(f: Factorization, rhs: np.ndarray) -> np.ndarray:
    """SPEC.md:320 solve_factored(f, rhs) -> x."""
    return f.solve(rhs)
