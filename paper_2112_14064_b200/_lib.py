"""ctypes binding of the C-ABI in include/rq_b200.h (librq_b200.so, built in-tree).

The library is the product: there is no Python or CPU fallback. Importing this
module fails loudly when the shared object is missing; numeric entry points
fail with RqError(code=2, config) when no sm_100a device is visible.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RQB_LIB: alternative build of the same library (development A/B runs only)
LIB_PATH = os.environ.get("RQB_LIB") or os.path.join(_HERE, "librq_b200.so")

# rq::errc (reference proj/include/rigaqep/types.hpp:14-23)
ERRC = {1: "generic", 2: "config", 3: "assembly", 4: "solver", 5: "verification",
        6: "domain", 7: "dimension", 8: "singular"}


class RqError(RuntimeError):
    """rq::Error equivalent (types.hpp:25-32): carries the errc code."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{ERRC.get(code, code)}] {msg}")
        self.code = code
        self.category = ERRC.get(code, "unknown")


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `make -C paper_2112_14064_b200` "
                      "(or __graft_entry__.build()); the B200 path has no fallback")

lib = C.CDLL(LIB_PATH)

i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
vp = C.c_void_p


def _nullable(base):
    """ndpointer argtype that also accepts None (NULL)."""
    class _N(base):
        @classmethod
        def from_param(cls, obj):
            return None if obj is None else base.from_param(obj)
    return _N


i32n, i64n, f64n = _nullable(i32p), _nullable(i64p), _nullable(f64p)


class SpaceDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("degree", C.c_int), ("elems", C.c_int),
                ("levels", C.c_int), ("alpha", C.c_double), ("beta", C.c_double)]


class SymbolicStats(C.Structure):
    _fields_ = [("n", C.c_int64), ("nfronts", C.c_int64), ("nlevels", C.c_int64),
                ("max_front", C.c_int64), ("max_npiv", C.c_int64), ("nnz_l", C.c_int64),
                ("nnz_u", C.c_int64), ("pool_doubles", C.c_int64), ("flops_lu", C.c_double),
                ("flops_schur", C.c_double), ("flops_schur_large", C.c_double),
                ("trisolve_bytes", C.c_double)]


class FactorInfo(C.Structure):
    _fields_ = [("swaps", C.c_int64), ("factor_ms", C.c_double), ("gflops", C.c_double),
                ("launches", C.c_int64)]


class OperatorOpts(C.Structure):
    _fields_ = [("sigma", C.c_double), ("scaling", C.c_int)]


class EigsOpts(C.Structure):
    _fields_ = [("nev", C.c_int), ("m", C.c_int), ("tol", C.c_double), ("seed", C.c_uint64),
                ("max_restarts", C.c_int), ("guard", C.c_int), ("profile", C.c_int), ("block", C.c_int)]


class GhOpts(C.Structure):
    _fields_ = [("nev", C.c_int), ("m", C.c_int), ("tol", C.c_double), ("seed", C.c_uint64),
                ("max_restarts", C.c_int)]


class GhInfo(C.Structure):
    _fields_ = [("nconv", C.c_int), ("cycles", C.c_int), ("restarts", C.c_int),
                ("lanczos_defect", C.c_double), ("sym_defect", C.c_double), ("launches", C.c_int64),
                ("t_total_ms", C.c_double)]


class EigsInfo(C.Structure):
    _fields_ = [("nconv", C.c_int), ("restarts", C.c_int), ("guard_passes", C.c_int),
                ("n_fa", C.c_int64), ("n_fb", C.c_int64), ("n_mv", C.c_int64),
                ("n_vv", C.c_int64), ("n_check", C.c_int64), ("n_restart", C.c_int64),
                ("macs_fa", C.c_double), ("macs_fb", C.c_double), ("macs_mv", C.c_double),
                ("macs_vv", C.c_double), ("macs_check", C.c_double),
                ("macs_restart", C.c_double), ("t_total_ms", C.c_double),
                ("t_factor_ms", C.c_double), ("t_solve_ms", C.c_double),
                ("t_spmv_ms", C.c_double), ("t_orth_ms", C.c_double), ("t_host_ms", C.c_double),
                ("launches", C.c_int64), ("restart_defect", C.c_double),
                ("t_ritz_ms", C.c_double), ("t_check_ms", C.c_double),
                ("t_restart_ms", C.c_double), ("t_sync_ms", C.c_double)]


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("rq_last_error", C.c_char_p)
_sig("rq_version", C.c_char_p)
_sig("rq_set_device", C.c_int, C.c_int)
_sig("rq_pencil_assemble", C.c_int, C.POINTER(SpaceDesc), C.POINTER(vp))
_sig("rq_pencil_assemble_acoustic", C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
     C.c_double, C.c_int, C.POINTER(vp))
_sig("rq_pencil_assemble_em", C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, vp, vp,
     C.POINTER(vp))
_sig("rq_pencil_assemble_device", C.c_int, C.POINTER(SpaceDesc), C.c_int, C.POINTER(vp), f64p)
_sig("rq_pencil_dims", C.c_int, vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64))
_sig("rq_pencil_csr", C.c_int, vp, i64n, i32n, f64n, f64n, f64n)
_sig("rq_pencil_supports", C.c_int, vp, i32n, i64n)
_sig("rq_pencil_destroy", None, vp)
_sig("rq_space_dims", C.c_int, C.POINTER(SpaceDesc), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
     C.POINTER(C.c_int64), C.POINTER(C.c_int64))
_sig("rq_space_boundary_mask", C.c_int, C.POINTER(SpaceDesc), vp, C.POINTER(C.c_int64))
_sig("rq_nd_order", C.c_int, C.c_int64, i32p, C.c_int, C.c_int, C.POINTER(vp))
_sig("rq_symbolic_stats_get", C.c_int, vp, C.POINTER(SymbolicStats))
_sig("rq_symbolic_perm", C.c_int, vp, i32p)
_sig("rq_symbolic_fronts", C.c_int, vp, i32p, i32p, i32p, i32p, i32p)
_sig("rq_symbolic_front_rows", C.c_int, vp, C.c_int64, i32p)
_sig("rq_symbolic_destroy", None, vp)
_sig("rq_factor_create", C.c_int, vp, C.c_int64, i64p, i32p, f64p, C.POINTER(vp))
_sig("rq_factor_refactor", C.c_int, vp, f64p)
_sig("rq_factor_get_info", C.c_int, vp, C.POINTER(FactorInfo))
_sig("rq_factor_solve", C.c_int, vp, f64p, f64p, C.c_int)
_sig("rq_factor_solve_ex", C.c_int, vp, f64p, f64p, C.c_int, C.c_int)
_sig("rq_factor_create_complex", C.c_int, vp, C.c_int64, i64p, i32p, f64p, vp, C.POINTER(vp))
_sig("rq_factor_refactor_complex", C.c_int, vp, f64p, vp, i64p, i32p)
_sig("rq_factor_solve_complex", C.c_int, vp, f64p, f64p, C.c_int)
_sig("rq_factor_front_export", C.c_int, vp, C.c_int64, vp, vp, C.POINTER(C.c_int64))
_sig("rq_factor_profile", C.c_int, vp, f64p, i64p, f64p)
_sig("rq_factor_dag_profile", C.c_int, vp, f64p)
_sig("rq_factor_bench_updcb", C.c_int, vp, C.c_int, C.c_int, f64p)
_sig("rq_factor_destroy", None, vp)
_sig("rq_mm_write", C.c_int, C.c_int64, i64p, i32p, f64p, f64n, C.c_char_p)
_sig("rq_mm_write_vector", C.c_int, C.c_int64, f64p, f64n, C.c_char_p)
_sig("rq_mm_read", C.c_int, C.c_char_p, C.POINTER(vp))
_sig("rq_mm_dims", C.c_int, vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int))
_sig("rq_mm_csr", C.c_int, vp, i64n, i32n, f64n, f64n)
_sig("rq_mm_destroy", None, vp)
_sig("rq_pencil_write_mm", C.c_int, vp, C.c_char_p)
_sig("rq_eigenpairs_json", C.c_int, C.c_int, f64n, f64n, f64n, C.c_char_p, C.c_int64, C.POINTER(C.c_int64))
_sig("rq_operator_create", C.c_int, C.c_int64, i64p, i32p, f64p, f64p, f64p, vp,
     C.POINTER(OperatorOpts), C.POINTER(vp))
_sig("rq_operator_create_pencil", C.c_int, vp, vp, C.POINTER(OperatorOpts), C.POINTER(vp))
_sig("rq_operator_varsigma", C.c_double, vp)
_sig("rq_operator_apply", C.c_int, vp, f64p, f64p)
_sig("rq_operator_b_inner", C.c_int, vp, f64p, f64p, C.POINTER(C.c_double))
_sig("rq_operator_spmv", C.c_int, vp, C.c_int, f64p, f64p)
_sig("rq_operator_arnoldi", C.c_int, vp, f64p, C.c_int, vp, vp)
_sig("rq_operator_factor", vp, vp)
_sig("rq_operator_destroy", None, vp)
_sig("rq_operator_time", C.c_int, vp, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double))
_sig("rq_eigs_run", C.c_int, vp, C.POINTER(EigsOpts), vp, vp, vp, vp, vp, C.POINTER(EigsInfo))
_sig("rq_eigs_ledger_json", C.c_int, vp, C.c_char_p, C.c_size_t)
_sig("rq_operator_ledger", C.c_int, vp, f64p)
_sig("rq_operator_release_workspace", C.c_int, vp)
_sig("rq_operator_ledger_json", C.c_int, vp, C.c_char_p, C.c_size_t)
_sig("rq_operator_ledger_reset", C.c_int, vp)
_sig("rq_scale_pencil", C.c_int, C.c_int64, f64p, f64p, f64p, C.POINTER(C.c_double), vp, vp)
_sig("rq_ritz_extract", C.c_int, f64p, C.c_int, C.c_double, C.c_double, vp, vp, vp, vp)
_sig("rq_operator_krylov_schur_restart", C.c_int, vp, C.c_int, C.c_int, f64p, f64p, C.POINTER(C.c_int))

_sig("rq_gh_create", C.c_int, C.c_int64, i64p, i32p, f64p, f64p, vp, C.c_double, C.POINTER(vp))
_sig("rq_gh_run", C.c_int, vp, C.POINTER(GhOpts), f64p, f64p, vp, C.POINTER(GhInfo))
_sig("rq_gh_destroy", None, vp)
_sig("rq_zeig_create", C.c_int, vp, C.c_int64, i64p, i32p, f64p, f64p, f64p, C.c_double, C.c_double,
     C.POINTER(vp))
_sig("rq_zeig_run", C.c_int, vp, C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_int, f64p, f64p, vp, i32p)
_sig("rq_zeig_destroy", None, vp)

# every symbol include/rq_b200.h declares (checked by tests/test_capi.py)
EXPORTS = [
    "rq_last_error", "rq_version", "rq_set_device", "rq_pencil_assemble", "rq_pencil_assemble_device",
    "rq_pencil_assemble_acoustic", "rq_pencil_assemble_em",
    "rq_pencil_dims", "rq_pencil_csr",
    "rq_pencil_supports", "rq_pencil_destroy", "rq_space_dims", "rq_space_boundary_mask",
    "rq_nd_order", "rq_symbolic_stats_get", "rq_symbolic_perm", "rq_symbolic_fronts",
    "rq_symbolic_front_rows", "rq_symbolic_destroy", "rq_factor_create", "rq_factor_refactor",
    "rq_factor_get_info", "rq_factor_solve", "rq_factor_solve_ex", "rq_factor_create_complex",
    "rq_factor_refactor_complex", "rq_factor_solve_complex", "rq_factor_front_export", "rq_factor_profile", "rq_factor_dag_profile", "rq_factor_bench_updcb",
    "rq_factor_destroy",
    "rq_operator_create", "rq_operator_create_pencil", "rq_mm_write", "rq_mm_write_vector", "rq_mm_read",
    "rq_mm_dims", "rq_mm_csr", "rq_mm_destroy", "rq_pencil_write_mm", "rq_eigenpairs_json", "rq_operator_varsigma", "rq_operator_apply", "rq_operator_b_inner",
    "rq_operator_spmv", "rq_operator_arnoldi", "rq_operator_factor", "rq_operator_destroy",
    "rq_operator_time",
    "rq_eigs_run", "rq_eigs_ledger_json", "rq_operator_ledger", "rq_operator_ledger_json", "rq_operator_release_workspace",
    "rq_operator_ledger_reset", "rq_scale_pencil", "rq_ritz_extract", "rq_operator_krylov_schur_restart",
    "rq_gh_create", "rq_gh_run", "rq_gh_destroy", "rq_zeig_create", "rq_zeig_run", "rq_zeig_destroy",
]


def check(rc: int) -> None:
    if rc != 0:
        raise RqError(rc, lib.rq_last_error().decode(errors="replace"))


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(vp)
