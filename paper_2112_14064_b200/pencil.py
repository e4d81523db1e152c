"""Input construction: rIGA/IGA vector spaces and the BASELINE quadratic pencil.

Mirrors the reference's space API (spaces.hpp:68-80: build_iga_space,
build_riga_space, boundary_mask) and SPEC's assembly module
with the BASELINE forms: K = int(div.div | curl.curl) + phi.phi, M = int phi.phi,
C = alpha M + beta K, (p+1)^2 Gauss points, constrained DOFs eliminated, one
shared CSR pattern (int64 rowptr, int32 col; sparse.hpp:16-47). Host C++ does
the work (csrc/host/spaces.cpp); this module only moves arrays.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import RqError, SpaceDesc, check

CURL, DIV = 0, 1  # rq::SpaceKind (spaces.hpp:30)


@dataclass
class QuadraticPencil:
    """K, C, M on one shared pattern over the free DOFs."""

    kind: int
    degree: int
    elems: int
    levels: int
    n_full: int
    n: int
    rowptr: np.ndarray
    col: np.ndarray
    K: np.ndarray
    C: np.ndarray
    M: np.ndarray
    box: np.ndarray            # (n, 4) inclusive element support boxes
    free_to_full: np.ndarray
    alpha: float = 0.05
    beta: float = 0.01
    meta: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    def q_values(self, sigma: float) -> np.ndarray:
        """Q(s) = K + s C + s^2 M entrywise (formed once on the host)."""
        return self.K + sigma * self.C + sigma * sigma * self.M

    def to_scipy(self, which: str = "K"):
        import scipy.sparse as sp
        vals = {"K": self.K, "C": self.C, "M": self.M}[which]
        return sp.csr_matrix((vals, self.col, self.rowptr), shape=(self.n, self.n))


def _desc(kind, degree, elems, levels, alpha=0.05, beta=0.01) -> SpaceDesc:
    return SpaceDesc(int(kind), int(degree), int(elems), int(levels), float(alpha), float(beta))


def space_dims(kind: int, degree: int, elems: int, levels: int = 0):
    """(nx, ny) of the x- and y-component tensor spaces."""
    d = _desc(kind, degree, elems, levels)
    out = [C.c_int64() for _ in range(4)]
    check(_lib.lib.rq_space_dims(C.byref(d), *[C.byref(o) for o in out]))
    return (out[0].value, out[1].value), (out[2].value, out[3].value)


def boundary_mask(kind: int, degree: int, elems: int, levels: int = 0) -> np.ndarray:
    """Constrained full-space DOF ids (em for curl, acoustic all-rigid for div)."""
    d = _desc(kind, degree, elems, levels)
    cnt = C.c_int64()
    check(_lib.lib.rq_space_boundary_mask(C.byref(d), None, C.byref(cnt)))
    out = np.zeros(cnt.value, dtype=np.int64)
    check(_lib.lib.rq_space_boundary_mask(C.byref(d), _lib.ptr(out), C.byref(cnt)))
    return out


def assemble(kind: int, degree: int, elems: int, levels: int = 0, alpha: float = 0.05,
             beta: float = 0.01) -> QuadraticPencil:
    """Assemble the BASELINE pencil (host C++, untimed input construction)."""
    d = _desc(kind, degree, elems, levels, alpha, beta)
    h = C.c_void_p()
    check(_lib.lib.rq_pencil_assemble(C.byref(d), C.byref(h)))
    try:
        nf, n, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        check(_lib.lib.rq_pencil_dims(h, C.byref(nf), C.byref(n), C.byref(nnz)))
        rowptr = np.zeros(n.value + 1, np.int64)
        col = np.zeros(nnz.value, np.int32)
        K = np.zeros(nnz.value)
        Cm = np.zeros(nnz.value)
        M = np.zeros(nnz.value)
        check(_lib.lib.rq_pencil_csr(h, rowptr, col, K, Cm, M))
        box = np.zeros(4 * n.value, np.int32)
        f2f = np.zeros(n.value, np.int64)
        check(_lib.lib.rq_pencil_supports(h, box, f2f))
    finally:
        _lib.lib.rq_pencil_destroy(h)
    return QuadraticPencil(kind, degree, elems, levels, nf.value, n.value, rowptr, col, K, Cm, M,
                           box.reshape(-1, 4), f2f, alpha, beta)


def baseline_config(name: str) -> QuadraticPencil:
    """The BASELINE.json configurations by short name."""
    table = {
        "cfg1": (DIV, 2, 32, 0), "cfg2_iga": (DIV, 3, 64, 0), "cfg2_riga": (DIV, 3, 64, 3),
        "cfg3_iga": (CURL, 4, 128, 0), "cfg3_riga": (CURL, 4, 128, 3),
        "cfg4_iga": (DIV, 3, 512, 0), "cfg4_riga": (DIV, 3, 512, 5),
    }
    # BASELINE configs[4] (cfg5): H(curl) 256^2, p = 2..5, IGA vs rIGA with C^0
    # separators every 8 elements (L = log2(256/8) = 5)
    for p in (2, 3, 4, 5):
        table[f"cfg5_p{p}_iga"] = (CURL, p, 256, 0)
        table[f"cfg5_p{p}_riga"] = (CURL, p, 256, 5)
    if name not in table:
        raise RqError(2, f"unknown config {name!r}")
    return assemble(*table[name])
