"""Wire formats over the C-ABI: Matrix Market files for
matrices and vectors, pencil export, and the eigenpair JSON dump.

Mirrors the reference's sparse module (sparse.hpp:141-146, sparse.cpp:121-174:
write_matrix_market / read_matrix_market / write_matrix_market_vector) and
SPEC.md:269 (pencil export), :503 (eigenpair dump {re, im, residual}).
"""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from . import _lib
from ._lib import check


def write_matrix_market(a, path: str) -> None:
    """a: (rowptr, col, values) CSR (values real or complex) or a scipy sparse
    matrix; coordinate real|complex general, 1-based, 17 significant digits."""
    if hasattr(a, "tocsr"):
        a = a.tocsr()
        rowptr, col, val = a.indptr, a.indices, a.data
    else:
        rowptr, col, val = a
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    val = np.asarray(val)
    re = np.ascontiguousarray(val.real, np.float64)
    im = np.ascontiguousarray(val.imag, np.float64) if np.iscomplexobj(val) else None
    check(_lib.lib.rq_mm_write(len(rowptr) - 1, rowptr, col, re, im, path.encode()))


def read_matrix_market(path: str):
    """(rowptr, col, values): sorted CSR, duplicates summed; values complex
    when the file is complex."""
    h = C.c_void_p()
    check(_lib.lib.rq_mm_read(path.encode(), C.byref(h)))
    try:
        n, nnz, cx = C.c_int64(), C.c_int64(), C.c_int()
        check(_lib.lib.rq_mm_dims(h, C.byref(n), C.byref(nnz), C.byref(cx)))
        rowptr = np.empty(n.value + 1, np.int64)
        col = np.empty(nnz.value, np.int32)
        re = np.empty(nnz.value)
        im = np.empty(nnz.value)
        check(_lib.lib.rq_mm_csr(h, rowptr, col, re, im))
    finally:
        _lib.lib.rq_mm_destroy(h)
    return rowptr, col, (re + 1j * im if cx.value else re)


def write_matrix_market_vector(x, path: str) -> None:
    """Dense vector as 'array complex general' (one "re im" per line)."""
    x = np.asarray(x)
    re = np.ascontiguousarray(x.real, np.float64)
    im = np.ascontiguousarray(x.imag, np.float64) if np.iscomplexobj(x) else None
    check(_lib.lib.rq_mm_write_vector(len(x), re, im, path.encode()))


def write_pencil(pencil, prefix: str) -> list[str]:
    """SPEC.md:269 pencil export: <prefix>K.mtx, <prefix>C.mtx, <prefix>M.mtx."""
    h = getattr(pencil, "handle", None)
    if h is not None:  # device-resident pencil: written from its own handle
        check(_lib.lib.rq_pencil_write_mm(h, prefix.encode()))
    else:
        for w in "KCM":
            write_matrix_market((pencil.rowptr, pencil.col, getattr(pencil, w)), prefix + w + ".mtx")
    return [prefix + w + ".mtx" for w in "KCM"]


def eigenpairs_json(pairs) -> str:
    """SPEC.md:503 eigenpair dump: JSON array of {re, im, residual}."""
    lam = np.array([complex(p.lam) for p in pairs])
    re = np.ascontiguousarray(lam.real)
    im = np.ascontiguousarray(lam.imag)
    res = np.ascontiguousarray([float(p.residual) for p in pairs], np.float64)
    n = C.c_int64()
    check(_lib.lib.rq_eigenpairs_json(len(lam), re, im, res, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(_lib.lib.rq_eigenpairs_json(len(lam), re, im, res, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def write_eigenpairs(pairs, path: str, vectors_prefix: str | None = None) -> None:
    """Eigenpair JSON and, optionally, each eigenvector as a Matrix Market
    dense vector <vectors_prefix><i>.mtx."""
    with open(path, "w") as f:
        f.write(eigenpairs_json(pairs))
    if vectors_prefix is not None:
        for i, p in enumerate(pairs):
            if p.u is not None:
                write_matrix_market_vector(p.u, f"{vectors_prefix}{i}.mtx")


def load_eigenpairs(path: str):
    """[(complex lambda, residual)] from an eigenpair JSON dump."""
    return [(complex(e["re"], e["im"]), float(e["residual"])) for e in json.load(open(path))]
