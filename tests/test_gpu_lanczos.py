"""GPU parity of solve_generalized_hermitian (SURVEY.md §8
row f4, the generalized-Hermitian Lanczos path): shift-invert Lanczos with
thick restarts on the device, against SPEC's known answers, dense LAPACK
(scipy.linalg.eigh) and the closed-form Maxwell eigenvalues of the unit
square (PAPER §6.4.1, Remark 2: the non-conductive problem reduces to the
generalized eigenproblem curl-curl u = lambda M u, lambda = pi^2 (i^2 + j^2)).

Tolerances: eigenvalues relative 1e-8 against LAPACK (both are converged to
residual 1e-10); the discrete Maxwell eigenvalue against the continuum value
at the discretisation error of p = 4 on 64^2 elements (relative 1e-3).
"""
import numpy as np
import pytest

import paper_2112_14064_b200 as rq

pytestmark = pytest.mark.gpu


def dense_pattern(n):
    rowptr = np.arange(0, n * n + 1, n, dtype=np.int64)
    col = np.tile(np.arange(n, dtype=np.int32), n)
    return rowptr, col, rq.Ordering(n, np.zeros((n, 4), np.int32), 1)


def test_known_answer_diag():
    """A = diag(1, 2, 3), B = I, s = 0 -> lambda = {1, 2, 3}."""
    rowptr, col, o = dense_pattern(3)
    A = np.diag([1.0, 2.0, 3.0]).ravel()
    B = np.eye(3).ravel()
    pairs = rq.solve_generalized_hermitian((rowptr, col, A), (rowptr, col, B), 0.0, 3, m=3, ordering=o)
    lam = sorted(p.lam.real for p in pairs)
    np.testing.assert_allclose(lam, [1.0, 2.0, 3.0], rtol=1e-12)
    assert all(p.lam.imag == 0 for p in pairs)


@pytest.mark.parametrize("s", [0.3, 7.5])
def test_dense_spd_pencil_vs_lapack(s):
    """A random symmetric A and SPD B (one dense front, 300 x 300): the nev
    eigenvalues nearest s equal LAPACK's; residuals and B-normalisation of the
    returned vectors recomputed on the host; the three-term structure of T
    holds to rounding (H_m symmetric tridiagonal)."""
    from scipy.linalg import eigh
    n, nev = 300, 8
    rng = np.random.default_rng(4)
    X = rng.standard_normal((n, n))
    A = (X + X.T) / 2 + 5 * np.eye(n)
    Y = rng.standard_normal((n, n))
    B = Y @ Y.T / n + np.eye(n)
    rowptr, col, o = dense_pattern(n)
    solver = rq.GeneralizedHermitianSolver(rowptr, col, A.ravel(), B.ravel(), s, o)
    pairs = solver.solve(nev, m=40, eps=1e-10, vectors=True, max_restarts=200)
    w = eigh(A, B, eigvals_only=True)
    ref = w[np.argsort(np.abs(w - s))][:nev]
    lam = np.array([p.lam.real for p in pairs])
    for x in lam:
        assert np.min(np.abs(ref - x)) <= 1e-8 * max(1.0, abs(x))
    for x in ref:
        assert np.min(np.abs(lam - x)) <= 1e-8 * max(1.0, abs(x))
    nA, nB = np.abs(A).sum(0).max(), np.abs(B).sum(0).max()
    for p in pairs:
        u = p.u
        r = A @ u - p.lam.real * (B @ u)
        assert np.linalg.norm(r) / ((nA + abs(p.lam) * nB) * np.linalg.norm(u)) <= 1e-10
        assert abs(np.linalg.norm(u) - 1.0) <= 1e-12
    info = solver.last_info
    assert info["lanczos_defect"] <= 1e-10 and info["sym_defect"] <= 1e-10


def test_maxwell_non_conductive_lambda_23_23():
    """PAPER §6.4.1: the non-conductive Maxwell problem on the unit square,
    p = 4, ne = 64 (H(curl) IGA), shift near 10442: the solver recovers
    lambda_{23,23} = pi^2 (23^2 + 23^2) = 10442.04 (A = curl-curl = K - M of
    the BASELINE pencil, whose K carries the extra phi.phi term; B = M). The
    nearest eigenvalues also match scipy's ARPACK shift-invert (an independent
    sparse eigensolver)."""
    import scipy.sparse.linalg as sla
    P = rq.assemble(rq.CURL, 4, 64, 0)
    A = P.K - P.M
    s = 10440.0
    pairs = rq.solve_generalized_hermitian(A, P.M, s, 4, pencil=P, eps=1e-10)
    lam = np.array([p.lam.real for p in pairs])
    exact = np.pi ** 2 * (23 ** 2 + 23 ** 2)
    assert abs(lam[0] - exact) <= 1e-3 * exact, (lam, exact)
    assert max(p.residual for p in pairs) <= 1e-10
    As = P.to_scipy("K") - P.to_scipy("M")
    Ms = P.to_scipy("M")
    w = sla.eigsh(As.tocsc(), k=4, M=Ms.tocsc(), sigma=s, which="LM", return_eigenvectors=False, tol=1e-12)
    w = np.sort(w[np.argsort(np.abs(w - s))])
    np.testing.assert_allclose(np.sort(lam), w, rtol=1e-8)


@pytest.mark.parametrize("ne,s", [(16, 200.0), (32, 1500.0)])
def test_maxwell_vs_oracle_restatement(ne, s):
    """GPU Lanczos against the oracle's restatement of
    solve_generalized_hermitian (complex multifrontal LU of A - s B on the
    reference kernels, Lanczos with full reorthogonalisation, thick restarts)
    on the H(curl) p = 4 Maxwell pencil: eigenvalues within relative 1e-9."""
    import oracle
    P = rq.assemble(rq.CURL, 4, ne, 0)
    pairs = rq.solve_generalized_hermitian(P.K - P.M, P.M, s, 6, pencil=P, eps=1e-10)
    lam = np.sort([p.lam.real for p in pairs])
    lo, ro = oracle.solve_generalized_hermitian(P.rowptr, P.col, P.K - P.M, P.M, P.box, P.elems, s, 6)
    assert np.all(ro <= 1e-10)
    np.testing.assert_allclose(lam, np.sort(lo), rtol=1e-9)
