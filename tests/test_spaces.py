"""Spaces, boundary masks, assembled pattern: pinned against the reference's own
spaces code (oracle/_ref, built from /root/reference) and the paper's numbers."""
import numpy as np
import pytest

import paper_2112_14064_b200 as rq
from paper_2112_14064_b200 import pencil as pen


def ref_or_skip():
    import oracle
    r = oracle.ref()
    if r is None:
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return r


def ref_space(kind, p, ne, L):
    import ctypes as C
    r = ref_or_skip()
    n = C.c_int64()
    nm = C.c_int64()
    assert r.ref_space(kind, p, ne, L, C.byref(n), None, None, C.byref(nm)) == 0
    box = np.zeros(4 * n.value, np.int32)
    mask = np.zeros(nm.value, np.int64)
    assert r.ref_space(kind, p, ne, L, C.byref(n), box.ctypes.data_as(C.c_void_p),
                       mask.ctypes.data_as(C.c_void_p), C.byref(nm)) == 0
    return n.value, box.reshape(-1, 4), mask


def full_pattern_nnz(box):
    # ordered pairs whose tensor supports share an element
    x0, x1, y0, y1 = (box[:, i][:, None] for i in range(4))
    ov = (x0 <= box[:, 1][None, :]) & (x1 >= box[:, 0][None, :]) & \
         (y0 <= box[:, 3][None, :]) & (y1 >= box[:, 2][None, :])
    return int(ov.sum())


def test_paper_dimensions():
    # PAPER.md:357,373 H(curl) p=4 ne=64: N = 9,112 (IGA), 10,804 (rIGA 16x16 macros)
    for L, N in ((0, 9112), (2, 10804)):
        (a, b), (c, d) = pen.space_dims(rq.CURL, 4, 64, L)
        assert a * b + c * d == N


@pytest.mark.parametrize("L,nnz", [(0, 1090240), (2, 1217968)])
def test_paper_pattern_nnz(L, nnz):
    # union pattern nnz of the full space
    n, box, _ = ref_space(0, 4, 64, L)
    assert full_pattern_nnz(box) == nnz


@pytest.mark.parametrize("kind,p,ne,L", [(rq.DIV, 2, 32, 0), (rq.DIV, 3, 16, 2), (rq.CURL, 4, 16, 1),
                                         (rq.CURL, 2, 8, 0), (rq.DIV, 3, 64, 3)])
def test_supports_and_mask_match_reference(kind, p, ne, L):
    n, box, mask = ref_space(kind, p, ne, L)
    assert np.array_equal(pen.boundary_mask(kind, p, ne, L), mask)
    P = rq.assemble(kind, p, ne, L)
    assert P.n_full == n and P.n == n - mask.size
    assert np.array_equal(P.box, box[P.free_to_full])
    assert np.array_equal(np.setdiff1d(np.arange(n), mask), P.free_to_full)


@pytest.mark.parametrize("name,nfull,nfree,nnz", [
    ("cfg1", 2244, 2112, 61628),
    ("cfg2_iga", 8844, 8580, 581976),
    ("cfg2_riga", 10804, 10512, 669308),
    ("cfg3_iga", 34584, 34060, 4195068),
    ("cfg3_riga", 42340, 41760, 4782956),
    ("cfg4_iga", 529420, 527364, 37227480),
    ("cfg4_riga", 595140, 592960, 40271308),
    ("cfg5_p2_iga", 132612, 131584, 4048380),
    ("cfg5_p2_riga", 132612, 131584, 4048380),  # p = 2: rIGA == IGA (App. B D4)
])
def test_config_sizes(name, nfull, nfree, nnz):
    P = rq.baseline_config(name)
    assert (P.n_full, P.n, P.nnz) == (nfull, nfree, nnz)


# SURVEY.md App. A (cfg5 = BASELINE configs[4], H(curl) 256^2, p = 2..5): N
# exact; pattern nnz, nnz(L), F_LU as printed there (3 / 3 / 2 significant
# digits); the largest front exact.
@pytest.mark.parametrize("name,nfull,nfree,nnz,nnzl,flu,maxf", [
    ("cfg5_p3_iga", 133644, 132612, 9.31e6, 51.9e6, 7.5e10, 1926),
    ("cfg5_p3_riga", 167620, 166464, 10.86e6, 33.2e6, 2.6e10, 1297),
    ("cfg5_p4_iga", 134680, 133644, 16.7e6, 86.1e6, 2.0e11, 2703),
    ("cfg5_p4_riga", 206724, 205440, 22.1e6, 46.2e6, 3.7e10, 1441),
    ("cfg5_p5_iga", 135720, 134680, 26.3e6, 128.2e6, 4.0e11, 3484),
    ("cfg5_p5_riga", 249924, 248512, 38.9e6, 62.6e6, 5.3e10, 1585),
])
def test_cfg5_sweep_sizes_and_symbolic(name, nfull, nfree, nnz, nnzl, flu, maxf):
    P = rq.baseline_config(name)
    assert (P.n_full, P.n) == (nfull, nfree)
    assert abs(P.nnz - nnz) <= 0.005 * nnz
    st = rq.nested_dissection_order(P).stats
    assert abs(st["nnz_l"] - nnzl) <= 0.0051 * nnzl
    assert abs(st["flops_lu"] - flu) <= 0.051 * flu
    assert st["max_front"] == maxf


def test_p2_riga_equals_iga():
    # at p=2 the separator rule is a no-op
    a = rq.assemble(rq.CURL, 2, 16, 0)
    b = rq.assemble(rq.CURL, 2, 16, 2)
    assert a.n == b.n and np.array_equal(a.col, b.col) and np.array_equal(a.K, b.K)


def test_assembly_properties(cfg1):
    import scipy.sparse as sp
    K, M, C = cfg1.to_scipy("K"), cfg1.to_scipy("M"), cfg1.to_scipy("C")
    assert abs(K - K.T).max() == 0.0 and abs(M - M.T).max() == 0.0
    assert abs(C - (0.05 * M + 0.01 * K)).max() < 1e-15 * abs(K).max()
    # M SPD: smallest eigenvalue positive (dense, small mesh)
    Ms = rq.assemble(rq.DIV, 2, 6).to_scipy("M").toarray()
    assert np.linalg.eigvalsh(Ms).min() > 0
    # sorted, unique column indices per row
    for r in range(0, cfg1.n, 97):
        c = cfg1.col[cfg1.rowptr[r]:cfg1.rowptr[r + 1]]
        assert np.all(np.diff(c) > 0)
    del sp


def _scipy_pencil_entries(kind, p, ne, L, P, stride=(3, 5)):
    """Independent scipy-BSpline quadrature of K, M for the space (kind, p, ne,
    L): knot vectors written from the reference's definition (open uniform
    knots; rIGA separators at the bisection breakpoints with multiplicity
    p - 1 in degree-p directions (C^1) and p - 1 in degree-(p-1) directions
    (C^0), spaces.cpp:12-77), an 8-point Gauss rule per element (exact for the
    polynomial integrands), curl = d(vy)/dx - d(vx)/dy, div = d(vx)/dx + d(vy)/dy."""
    from scipy.interpolate import BSpline
    seps = sorted({b * (ne >> l) for l in range(1, L + 1) for b in range(1, 1 << l, 2)})

    def knots(deg, cont):
        t = list(np.zeros(deg + 1))
        for b in range(1, ne):
            t += [b / ne] * ((deg - cont) if b in seps else 1)
        return np.array(t + [1.0] * (deg + 1))

    def basis(deg, cont):
        t = knots(deg, cont)
        nb = len(t) - deg - 1
        return [BSpline(t, np.eye(nb)[i], deg, extrapolate=False) for i in range(nb)]

    hi, lo = basis(p, 1), basis(p - 1, 0)
    g, w = np.polynomial.legendre.leggauss(8)
    xs = np.concatenate([e / ne + (g + 1) / (2 * ne) for e in range(ne)])
    ws = np.concatenate([w / (2 * ne) for e in range(ne)])

    def ev(bs, x, d=0):
        return np.array([np.nan_to_num((bb.derivative(d) if d else bb)(x)) for bb in bs])

    H, Hd, Lo, Lod = ev(hi, xs), ev(hi, xs, 1), ev(lo, xs), ev(lo, xs, 1)
    # DOF numbering: x-component first, x index fastest (spaces.hpp:33,62-63)
    if kind == rq.DIV:   # x-comp hi(x) lo(y), y-comp lo(x) hi(y)
        cx, cy = (H, Hd, Lo, Lod), (Lo, Lod, H, Hd)
    else:                # curl: x-comp lo(x) hi(y), y-comp hi(x) lo(y)
        cx, cy = (Lo, Lod, H, Hd), (H, Hd, Lo, Lod)
    phis = [("x", i, j) for j in range(len(cx[2])) for i in range(len(cx[0]))]
    phis += [("y", i, j) for j in range(len(cy[2])) for i in range(len(cy[0]))]
    W = np.outer(ws, ws)  # [x, y]

    def fields(ph):
        c, i, j = ph
        bx, dbx, by, dby = cx if c == "x" else cy
        v = np.outer(bx[i], by[j])
        dx, dy = np.outer(dbx[i], by[j]), np.outer(bx[i], dby[j])
        z = np.zeros_like(v)
        if kind == rq.DIV:
            return (v, z, dx) if c == "x" else (z, v, dy)
        return (v, z, -dy) if c == "x" else (z, v, dx)

    F = [fields(phis[g_]) for g_ in P.free_to_full]
    Kd, Md = P.to_scipy("K").toarray(), P.to_scipy("M").toarray()
    worst = 0.0
    for a in range(0, P.n, stride[0]):
        for b in range(0, P.n, stride[1]):
            m = np.sum(W * (F[a][0] * F[b][0] + F[a][1] * F[b][1]))
            k = np.sum(W * F[a][2] * F[b][2]) + m
            worst = max(worst, abs(Md[a, b] - m) / np.abs(Md).max(), abs(Kd[a, b] - k) / np.abs(Kd).max())
    return worst


@pytest.mark.parametrize("kind,p,ne,L", [(rq.DIV, 2, 4, 0), (rq.DIV, 3, 8, 1), (rq.CURL, 3, 8, 0),
                                         (rq.CURL, 4, 8, 1), (rq.CURL, 5, 8, 1)])
def test_assembly_against_independent_quadrature(kind, p, ne, L):
    """K, M vs an independent scipy-BSpline assembly: H(div) and H(curl),
    p = 2..5, IGA and rIGA (SPEC.md:233 independent-quadrature oracle)."""
    P = rq.assemble(kind, p, ne, L)
    assert _scipy_pencil_entries(kind, p, ne, L, P) <= 1e-13


@pytest.mark.parametrize("name", ["cfg1", "cfg2_iga", "cfg2_riga", "cfg3_iga", "cfg3_riga", "cfg5_p3_riga"])
def test_assembly_against_reference_spaces(name):
    """The product's pencil vs oracle/ref_assembly.cpp, which assembles on the
    reference's own build_*_space / boundary_mask / eval_basis_derivatives /
    piola_map (compiled from /root/reference): identical pattern and support
    boxes, values to rounding (different summation order)."""
    import oracle
    ref_or_skip()
    R = oracle.ref_config(name)
    P = rq.baseline_config(name)
    assert (R.n_full, R.n, R.nnz) == (P.n_full, P.n, P.nnz)
    assert np.array_equal(R.rowptr, P.rowptr) and np.array_equal(R.col, P.col)
    assert np.array_equal(R.box, P.box)
    for w in "KCM":
        a, b = getattr(P, w), getattr(R, w)
        scale = np.abs(b).max()
        assert np.abs(a - b).max() <= 1e-14 * scale
        big = np.abs(b) > 1e-6 * scale
        assert np.max(np.abs(a - b)[big] / np.abs(b)[big]) <= 1e-11
