"""ORACLE — TEST INFRASTRUCTURE ONLY. The reference's own Matrix Market
writers / reader (sparse.cpp:121-174, in oracle/_ref/liboracle_ref.so) run in
a child interpreter that never imports numpy: the reference's iostream code
crashes in a process that has numpy's bundled runtime libraries loaded, while
it runs fine from plain C / ctypes. Arrays travel as raw files."""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile

import numpy as np

from . import REF_PATH

_CHILD = r'''
import array, ctypes as C, sys
lib = C.CDLL(sys.argv[1])
op, d = sys.argv[2], sys.argv[3]
def load(name, code):
    a = array.array(code)
    with open(d + "/" + name, "rb") as f:
        a.frombytes(f.read())
    return a
def buf(a, ct):
    return (ct * len(a)).from_buffer(a) if len(a) else None
if op == "write":
    rp, col, re = load("rp", "q"), load("col", "i"), load("re", "d")
    im = load("im", "d") if sys.argv[5] == "1" else None
    rc = lib.ref_mm_write(C.c_int64(len(rp) - 1), buf(rp, C.c_int64), buf(col, C.c_int32), buf(re, C.c_double),
                          buf(im, C.c_double) if im is not None else None, sys.argv[4].encode())
elif op == "vector":
    re = load("re", "d")
    im = load("im", "d") if sys.argv[5] == "1" else None
    rc = lib.ref_mm_write_vector(C.c_int64(len(re)), buf(re, C.c_double),
                                 buf(im, C.c_double) if im is not None else None, sys.argv[4].encode())
else:
    n, nnz = C.c_int64(), C.c_int64()
    rc = lib.ref_mm_read(sys.argv[4].encode(), C.byref(n), C.byref(nnz), None, None, None, None)
    if rc == 0:
        rp = array.array("q", [0] * (n.value + 1)); col = array.array("i", [0] * max(nnz.value, 1))
        re = array.array("d", [0.0] * max(nnz.value, 1)); im = array.array("d", [0.0] * max(nnz.value, 1))
        rc = lib.ref_mm_read(sys.argv[4].encode(), C.byref(n), C.byref(nnz), buf(rp, C.c_int64),
                             buf(col, C.c_int32), buf(re, C.c_double), buf(im, C.c_double))
        for name, a in (("rp", rp), ("col", col[:nnz.value]), ("re", re[:nnz.value]), ("im", im[:nnz.value])):
            with open(d + "/" + name, "wb") as f:
                a.tofile(f)
sys.exit(rc)
'''


def _child(op: str, d: str, *args: str) -> None:
    subprocess.run([sys.executable, "-c", _CHILD, REF_PATH, op, d, *args], check=True)


def available() -> bool:
    return os.path.exists(REF_PATH)


def write(rowptr, col, re, im, path: str) -> None:
    with tempfile.TemporaryDirectory() as d:
        np.ascontiguousarray(rowptr, np.int64).tofile(d + "/rp")
        np.ascontiguousarray(col, np.int32).tofile(d + "/col")
        np.ascontiguousarray(re, np.float64).tofile(d + "/re")
        if im is not None:
            np.ascontiguousarray(im, np.float64).tofile(d + "/im")
        _child("write", d, path, "1" if im is not None else "0")


def write_vector(re, im, path: str) -> None:
    with tempfile.TemporaryDirectory() as d:
        np.ascontiguousarray(re, np.float64).tofile(d + "/re")
        if im is not None:
            np.ascontiguousarray(im, np.float64).tofile(d + "/im")
        _child("vector", d, path, "1" if im is not None else "0")


def read(path: str):
    with tempfile.TemporaryDirectory() as d:
        _child("read", d, path)
        return (np.fromfile(d + "/rp", np.int64), np.fromfile(d + "/col", np.int32),
                np.fromfile(d + "/re", np.float64), np.fromfile(d + "/im", np.float64))
