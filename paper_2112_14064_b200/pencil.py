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


class DevicePencil(QuadraticPencil):
    """A device-assembled pencil whose K, C, M stay in HBM.

    The pattern, supports and numbering are on the host as usual; K, C, M are
    copied to host arrays on first access only. build_operator uses the
    device values in place (rq_operator_create_pencil)."""

    device_resident = True

    def __init__(self, handle, **kw):
        self._handle = handle
        self._vals = {}
        super().__init__(K=None, C=None, M=None, **kw)

    def _get(self, which):
        if which not in self._vals:
            arrs = {w: np.empty(self.nnz) for w in "KCM"}
            check(_lib.lib.rq_pencil_csr(self._handle, None, None, arrs["K"], arrs["C"], arrs["M"]))
            self._vals.update(arrs)
        return self._vals[which]

    K = property(lambda self: self._get("K"), lambda self, v: None)
    C = property(lambda self: self._get("C"), lambda self, v: None)
    M = property(lambda self: self._get("M"), lambda self, v: None)

    @property
    def handle(self):
        return self._handle

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value and _lib is not None and _lib.lib is not None:  # (interpreter shutdown)
            _lib.lib.rq_pencil_destroy(h)
            self._handle = None


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
             beta: float = 0.01, device: bool = False, resident: bool = False,
             stage_ms=None) -> QuadraticPencil:
    """Assemble the BASELINE pencil: host C++ (default) or, with device=True,
    on the current CUDA device (bit-identical result; stage_ms, a float64
    array of 5, receives the device ms of pattern / element / gather and the
    host ms of the O(n) preparation and of the copy back). resident=True
    (device only) returns a DevicePencil whose K, C, M stay in HBM."""
    d = _desc(kind, degree, elems, levels, alpha, beta)
    h = C.c_void_p()
    if resident and not device:
        raise RqError(2, "resident=True needs device=True")
    if device:
        ms = np.zeros(5) if stage_ms is None else stage_ms
        check(_lib.lib.rq_pencil_assemble_device(C.byref(d), 1 if resident else 0, C.byref(h), ms))
    else:
        check(_lib.lib.rq_pencil_assemble(C.byref(d), C.byref(h)))
    if resident:
        try:
            nf, n, nnz = C.c_int64(), C.c_int64(), C.c_int64()
            check(_lib.lib.rq_pencil_dims(h, C.byref(nf), C.byref(n), C.byref(nnz)))
            rowptr = np.empty(n.value + 1, np.int64)
            col = np.empty(nnz.value, np.int32)
            check(_lib.lib.rq_pencil_csr(h, rowptr, col, None, None, None))
            box = np.empty(4 * n.value, np.int32)
            f2f = np.empty(n.value, np.int64)
            check(_lib.lib.rq_pencil_supports(h, box, f2f))
        except Exception:
            _lib.lib.rq_pencil_destroy(h)
            raise
        return DevicePencil(h, kind=kind, degree=degree, elems=elems, levels=levels, n_full=nf.value,
                            n=n.value, rowptr=rowptr, col=col, box=box.reshape(-1, 4),
                            free_to_full=f2f, alpha=alpha, beta=beta)
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


ACOUSTIC_EDGES = {"left": 1, "right": 2, "bottom": 4, "top": 8}


def assemble_acoustic(degree: int, elems: int, levels: int = 0, rho: float = 1.0, c: float = 340.0,
                      alpha: float = 5e4, beta: float = 200.0, absorbing=("top",)) -> QuadraticPencil:
    """The paper's vibroacoustic pencil (SPEC.md:225 assemble_acoustic; PAPER.md:165-200,
    the Fig. 8 cavity: unit square, one absorbing wall, air rho = 1, c = 340, impedance
    alpha = 5e4, beta = 200): K = rho c^2 div-div + alpha edge term, C = beta edge term,
    M = rho mass; rigid edges constrained, absorbing ones free. Real pencil."""
    mask = 0
    for e in absorbing:
        mask |= ACOUSTIC_EDGES[e]
    h = C.c_void_p()
    check(_lib.lib.rq_pencil_assemble_acoustic(int(degree), int(elems), int(levels), float(rho), float(c),
                                               float(alpha), float(beta), int(mask), C.byref(h)))
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
    return QuadraticPencil(DIV, degree, elems, levels, nf.value, n.value, rowptr, col, K, Cm, M,
                           box.reshape(-1, 4), f2f, 0.0, 0.0)


def assemble_em(degree: int, elems: int, levels: int = 0, mu: float = 1.0, eps: float = 1.0,
                layers=((0.0, 1.0, 1.0, 1.0),)) -> QuadraticPencil:
    """The paper's conductive electromagnetic pencil (SPEC.md:216-224 assemble_em;
    PAPER.md §2.1): K = -(1/mu) curl-curl, M = eps mass, C = -i D with D the
    conductivity-weighted mass over horizontal layers (y0, y1, sigma_x, sigma_y).
    The returned pencil's C is complex (purely imaginary): solve it with
    solve_quadratic_complex."""
    lay = np.ascontiguousarray(np.asarray(layers, np.float64).reshape(-1, 4))
    h = C.c_void_p()
    check(_lib.lib.rq_pencil_assemble_em(int(degree), int(elems), int(levels), float(mu), float(eps), len(lay),
                                         _lib.ptr(lay.reshape(-1)), None, C.byref(h)))
    try:
        nf, n, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        check(_lib.lib.rq_pencil_dims(h, C.byref(nf), C.byref(n), C.byref(nnz)))
        rowptr = np.zeros(n.value + 1, np.int64)
        col = np.zeros(nnz.value, np.int32)
        K = np.zeros(nnz.value)
        D = np.zeros(nnz.value)
        M = np.zeros(nnz.value)
        check(_lib.lib.rq_pencil_csr(h, rowptr, col, K, D, M))
        box = np.zeros(4 * n.value, np.int32)
        f2f = np.zeros(n.value, np.int64)
        check(_lib.lib.rq_pencil_supports(h, box, f2f))
    finally:
        _lib.lib.rq_pencil_destroy(h)
    return QuadraticPencil(CURL, degree, elems, levels, nf.value, n.value, rowptr, col, K, -1j * D, M,
                           box.reshape(-1, 4), f2f, 0.0, 0.0)


def baseline_config(name: str, device: bool = False, resident: bool = False) -> QuadraticPencil:
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
    return assemble(*table[name], device=device, resident=resident)
