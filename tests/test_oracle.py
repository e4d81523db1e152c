"""Pinning the oracle: SPEC known answers, the reference's own kernels (oracle/_ref),
and independent dense solves (numpy/scipy). CPU only."""
import numpy as np
import pytest

import oracle
import paper_2112_14064_b200 as rq


class Tiny:
    """A dense n x n 'pencil' on one front (box/elems chosen so ND makes one leaf)."""

    def __init__(self, K, C=None, M=None):
        K = np.atleast_2d(np.asarray(K, dtype=complex))
        n = K.shape[0]
        C = np.zeros_like(K) if C is None else np.atleast_2d(np.asarray(C, dtype=complex))
        M = np.eye(n, dtype=complex) if M is None else np.atleast_2d(np.asarray(M, dtype=complex))
        self.n, self.elems = n, 1
        self.rowptr = np.arange(0, n * n + 1, n, dtype=np.int64)
        self.col = np.tile(np.arange(n, dtype=np.int32), n)
        self.K, self.C, self.M = K.ravel(), C.ravel(), M.ravel()
        self.box = np.zeros((n, 4), np.int32)


def test_lu_known_answer_3x3():
    # [[4,3,0],[6,3,1],[0,1,2]] by hand elimination with threshold 0.1:
    # |4| >= 0.1*6 keeps the diagonal: l21 = 1.5, u22 = 3 - 4.5 = -1.5, ...
    A = np.array([[4, 3, 0], [6, 3, 1], [0, 1, 2]], float)
    t = Tiny(A)
    f = oracle.Factor(3, t.rowptr, t.col, A.ravel(), t.box, 1)
    F, ipiv, rows = f.front(0, 3, 3)
    assert list(ipiv) == [0, 1, 2] and f.swaps == 0
    L = np.tril(F.real, -1) + np.eye(3)
    U = np.triu(F.real)
    np.testing.assert_allclose(L, [[1, 0, 0], [1.5, 1, 0], [0, -2 / 3, 1]], atol=1e-14)
    np.testing.assert_allclose(U, [[4, 3, 0], [0, -1.5, 1], [0, 0, 2 + 2 / 3]], atol=1e-14)
    x = f.solve(np.array([1.0, 2.0, 3.0]))
    np.testing.assert_allclose(A @ x.real, [1, 2, 3], atol=1e-14)


def test_lu_identity_and_pivoting():
    t = Tiny(np.eye(4))
    f = oracle.Factor(4, t.rowptr, t.col, np.eye(4).ravel(), t.box, 1)
    assert f.fa_macs == 0  # identity -> fa increment 0
    A = np.array([[1e-3, 1.0], [1.0, 1.0]])
    f = oracle.Factor(2, Tiny(A).rowptr, Tiny(A).col, A.ravel(), np.zeros((2, 4), np.int32), 1)
    _, ipiv, _ = f.front(0, 2, 2)
    assert list(ipiv) == [1, 1] and f.swaps == 1  # |1e-3| < 0.1 * 1 -> swap


def test_spd_50_solve_residual():
    # SPEC.md:327 random SPD 50x50: ||Ax - b|| / ||b|| <= 1e-12
    rng = np.random.default_rng(0)
    B = rng.standard_normal((50, 50))
    A = B @ B.T + 50 * np.eye(50)
    t = Tiny(A)
    f = oracle.Factor(50, t.rowptr, t.col, A.ravel(), t.box, 1)
    b = rng.standard_normal(50)
    x = f.solve(b).real
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) <= 1e-12


def test_scalar_qep():
    # (K, C, M) = (2, 3, 1) -> lambda = -1, -2
    t = Tiny([[2.0]], [[3.0]], [[1.0]])
    E = oracle.Eig(t, 0.0, leaf=64)
    lam, res = E.solve_quadratic(2, m=2, tol=1e-12)
    assert sorted(np.round(lam.real, 12)) == [-2.0, -1.0] and np.all(np.abs(lam.imag) < 1e-12)


def test_2x2_qep():
    # K = diag(1,4), C = 0, M = I, s = 0.1 -> +-i, +-2i (nearest 2: +-i)
    t = Tiny(np.diag([1.0, 4.0]))
    E = oracle.Eig(t, 0.1)
    lam, res = E.solve_quadratic(2, m=3, tol=1e-12)
    np.testing.assert_allclose(sorted(lam.imag), [-1, 1], atol=1e-10)
    np.testing.assert_allclose(lam.real, 0, atol=1e-10)


def test_operator_against_dense_linearisation():
    """apply_operator vs the dense 2N x 2N (A - sB)^{-1} B."""
    rng = np.random.default_rng(3)
    n = 6
    K = rng.standard_normal((n, n)); K = K + K.T + 8 * np.eye(n)
    C = rng.standard_normal((n, n)); C = C + C.T
    M = rng.standard_normal((n, n)); M = M @ M.T + n * np.eye(n)
    s = 0.37
    t = Tiny(K, C, M)
    E = oracle.Eig(t, s)
    v = rng.standard_normal(2 * n)
    r = E.apply(v)
    # linearisation A z = lam B z with z = (u, lam u): A = [[-C, -K],[I, 0]]... use the block formula
    Q = K + s * C + s * s * M
    ru = -np.linalg.solve(Q, s * M @ v[:n] + C @ v[:n] + M @ v[n:])
    rl = s * ru + v[:n]
    np.testing.assert_allclose(r.real, np.r_[ru, rl], rtol=1e-10, atol=1e-12)
    # eigen-consistency: S (u; lam u) = theta (u; lam u), theta = 1/(lam - s)
    from scipy.linalg import eig
    Z = np.zeros((n, n)); I = np.eye(n)
    Al = np.block([[Z, I], [-K, -C]]); Bl = np.block([[I, Z], [Z, M]])
    w, X = eig(Al, Bl)
    lam = w[0]; u = X[:n, 0]
    z = np.r_[u, lam * u]
    rz = E.apply(z)
    np.testing.assert_allclose(rz, z / (lam - s), rtol=1e-8, atol=1e-10)


def test_kernels_match_reference_build():
    """Restated kern:: (liboracle.so) vs the reference's own kernels.cpp /
    kernels_avx2.cpp compiled from /root/reference (oracle/_ref)."""
    r = oracle.ref()
    if r is None:
        pytest.skip("oracle/_ref not built")
    port = oracle.port()
    rng = np.random.default_rng(5)
    n = 300
    A = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * (rng.random((n, n)) < 0.05)
    import scipy.sparse as sp
    S = sp.csr_matrix(A)
    S.sort_indices()
    rp, col = S.indptr.astype(np.int64), S.indices.astype(np.int32)
    val = oracle.cplx(S.data)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    for backend in (b"scalar", b"avx2"):
        if r.ref_select_backend(backend) != 0:
            continue
        y1, y2 = np.zeros(2 * n), np.zeros(2 * n)
        port.oracle_kern_spmv(n, rp, col, val, oracle.cplx(x), y1)
        r.ref_kern_spmv(n, rp, col, val, oracle.cplx(x), y2)
        tol = 0 if backend == b"scalar" else 1e-14
        assert np.max(np.abs(y1 - y2)) <= tol * max(1, np.max(np.abs(y1)))
        d1, d2 = np.zeros(2), np.zeros(2)
        port.oracle_kern_dotc(oracle.cplx(x), oracle.cplx(x[::-1].copy()), n, d1)
        r.ref_kern_dotc(oracle.cplx(x), oracle.cplx(x[::-1].copy()), n, d2)
        assert np.max(np.abs(d1 - d2)) <= tol * np.max(np.abs(d1)) + 0
        # elim_step: 6-argument rank-1 update, zero multipliers skipped
        tile = rng.standard_normal((8, 10)) + 0j
        lcol = np.array([1, 0, 2, 0, 0, 1j, 3, 0], complex)
        urow = rng.standard_normal(10) + 1j
        t1, t2 = oracle.cplx(tile), oracle.cplx(tile)
        m1 = port.oracle_kern_elim(t1, 10, oracle.cplx(lcol), oracle.cplx(urow), 8, 10)
        m2 = r.ref_kern_elim(t2, 10, oracle.cplx(lcol), oracle.cplx(urow), 8, 10)
        assert m1 == m2 == 4 * 10
        assert np.max(np.abs(t1 - t2)) <= 1e-14
    r.ref_select_backend(b"auto")


def test_oracle_port_vs_reference_kernel_build(cfg1):
    r = oracle.ref()
    if r is None:
        pytest.skip("oracle/_ref not built")
    a = oracle.Eig(cfg1, -0.5, kind="port")
    b = oracle.Eig(cfg1, -0.5, kind="reference")
    v = np.random.default_rng(0).uniform(-1, 1, 2 * cfg1.n)
    ra, rb = a.apply(v), b.apply(v)
    assert np.max(np.abs(ra - rb)) <= 1e-12 * np.max(np.abs(ra))


def test_oracle_eigs_vs_scipy_dense():
    """Non-degenerate pencil (C perturbed by a diagonal): oracle Krylov-Schur vs
    scipy's dense QZ on the companion linearisation."""
    from scipy.linalg import eigvals
    P = rq.assemble(rq.DIV, 2, 6, 0)
    rng = np.random.default_rng(11)
    C = P.C.copy()
    diag = np.array([np.searchsorted(P.col[P.rowptr[i]:P.rowptr[i + 1]], i) + P.rowptr[i]
                     for i in range(P.n)])
    C[diag] += 0.5 * rng.random(P.n) * P.M[diag]
    sigma = -0.5
    E = oracle.Eig(P, sigma, C_=C)
    lam, res = E.solve_quadratic(6, tol=1e-10, max_restarts=400)
    assert np.all(res <= 1e-10)
    Kd = P.to_scipy("K").toarray(); Md = P.to_scipy("M").toarray()
    Cd = P.to_scipy("M").toarray() * 0
    import scipy.sparse as sp
    Cd = sp.csr_matrix((C, P.col, P.rowptr), shape=(P.n, P.n)).toarray()
    n = P.n
    Z, I = np.zeros((n, n)), np.eye(n)
    w = eigvals(np.block([[Z, I], [-Kd, -Cd]]), np.block([[I, Z], [Z, Md]]))
    w = w[np.argsort(np.abs(w - sigma))][:6]
    for x in lam:
        assert np.min(np.abs(w - x)) <= 1e-8 * abs(x)


def test_oracle_cluster_closed_form(cfg1):
    """all requested pairs are copies of -0.03 +- i sqrt(0.9991)."""
    E = oracle.Eig(cfg1, -0.5)
    lam, res = E.solve_quadratic(10, tol=1e-10)
    ref = -0.03 + 1j * np.sqrt(0.9991)
    assert np.all(np.minimum(np.abs(lam - ref), np.abs(lam - np.conj(ref))) <= 1e-8)
    assert np.sum(lam.imag > 0) == 5 and np.all(res <= 1e-10)
    assert E.ledger["fa"]["ops"] == 1


def test_scale_pencil_known_answer():
    """K = 4I, C = M = I -> varsigma = 2, scaled pencil (4I, 2I, 4I);
    roots of 4 + 2 gamma + 4 gamma^2 are those of 4 + lambda + lambda^2 over 2."""
    n = 3
    rp = np.arange(n + 1, dtype=np.int64)
    col = np.arange(n, dtype=np.int32)
    vs, Cs, Ms = oracle.scale_pencil(n, rp, col, 4 * np.ones(n), np.ones(n), np.ones(n))
    assert vs == 2.0
    assert np.array_equal(Cs, 2 * np.ones(n)) and np.array_equal(Ms, 4 * np.ones(n))
    g = np.sort_complex(np.roots([4, 2, 4]))
    lam = np.sort_complex(np.roots([1, 1, 4]))
    assert np.allclose(2 * g, lam, rtol=1e-14)
    # equal norms -> varsigma = 1, pencil unchanged
    vs1, C1, M1 = oracle.scale_pencil(n, rp, col, np.ones(n), 3 * np.ones(n), np.ones(n))
    assert vs1 == 1.0 and np.array_equal(C1, 3 * np.ones(n))
    with pytest.raises(oracle.OracleError) as e:  # zero M
        oracle.scale_pencil(n, rp, col, np.ones(n), np.ones(n), np.zeros(n))
    assert e.value.code == 6


def test_oracle_generalized_hermitian_known_answers():
    """The oracle's solve_generalized_hermitian: diag(1, 2, 3)
    with B = I -> {1, 2, 3}, and the H(curl) p = 4 16^2 Maxwell
    pencil (curl-curl = K - M, B = M) against scipy's ARPACK shift-invert; the
    double eigenvalue pi^2 (2^2 + 4^2) = 197.39 within the discretisation error."""
    import scipy.sparse.linalg as sla
    rp = np.arange(0, 10, 3, dtype=np.int64)
    col = np.tile(np.arange(3, dtype=np.int32), 3)
    lam, res = oracle.solve_generalized_hermitian(rp, col, np.diag([1.0, 2, 3]).ravel(), np.eye(3).ravel(),
                                                  np.zeros((3, 4), np.int32), 1, 0.0, 3, m=3)
    np.testing.assert_allclose(np.sort(lam), [1, 2, 3], rtol=1e-13)
    P = rq.assemble(rq.CURL, 4, 16, 0)
    lam, res = oracle.solve_generalized_hermitian(P.rowptr, P.col, P.K - P.M, P.M, P.box, P.elems, 200.0, 4)
    assert np.all(res <= 1e-10)
    w = sla.eigsh((P.to_scipy("K") - P.to_scipy("M")).tocsc(), k=4, M=P.to_scipy("M").tocsc(), sigma=200.0,
                  return_eigenvectors=False, tol=1e-12)
    np.testing.assert_allclose(np.sort(lam), np.sort(w), rtol=1e-9)
    assert abs(lam[0] - 20 * np.pi ** 2) <= 1e-4 * 20 * np.pi ** 2
