"""Complex shifts and complex pencils on the B200 path (
SPEC.md:408-470 over complex scalars; "Complex shift support: Q(s) complex
non-symmetric handled by the pivoting LU"): complex Krylov-Schur on the
device with the real-equivalent complex LU.

Known answers: scipy's dense QZ on the companion linearisation (non-degenerate
pencil, complex shift); the conductive Maxwell pencil with uniform
conductivity, K = -curl-curl, C = -i sigma M, M = mass (SPEC.md:216-224 sign
convention), whose eigenvalues are lam = i sigma / 2 +- sqrt(kappa - sigma^2 / 4)
for every generalized eigenvalue kappa of (curl-curl, M) (from ARPACK), and
the gyroscopic symmetry lam -> -conj(lam).
"""
import numpy as np
import pytest

import paper_2112_14064_b200 as rq

pytestmark = pytest.mark.gpu


def _perturbed(ne=8):
    P = rq.assemble(rq.DIV, 2, ne, 0)
    diag = np.array([P.rowptr[i] + np.searchsorted(P.col[P.rowptr[i]:P.rowptr[i + 1]], i)
                     for i in range(P.n)])
    rng = np.random.default_rng(11)
    P.C = P.C.copy()
    P.C[diag] += 0.5 * rng.random(P.n) * P.M[diag]
    return P


@pytest.mark.parametrize("s", [-0.2 + 0.7j, -0.5 + 0.0j, -0.05 - 1.2j])
def test_complex_shift_vs_dense_qz(s):
    from scipy.linalg import eigvals
    P = _perturbed()
    nev = 6
    pairs = rq.solve_quadratic_complex(P, s, nev, m=30, eps=1e-10, max_restarts=300, vectors=True)
    lam = np.array([p.lam for p in pairs])
    assert max(p.residual for p in pairs) <= 1e-10
    n = P.n
    Kd, Cd, Md = (P.to_scipy(w).toarray() for w in "KCM")
    Z, I = np.zeros((n, n)), np.eye(n)
    w = eigvals(np.block([[Z, I], [-Kd, -Cd]]), np.block([[I, Z], [Z, Md]]))
    w = w[np.argsort(np.abs(w - s))][:nev]
    for x in lam:
        assert np.min(np.abs(w - x)) <= 1e-8 * abs(x)
    for x in w:
        assert np.min(np.abs(lam - x)) <= 1e-8 * abs(x)
    nrm = lambda A: abs(A).sum(0).max()  # noqa: E731
    for p in pairs:
        r = Kd @ p.u + p.lam * (Cd @ p.u) + p.lam ** 2 * (Md @ p.u)
        den = (nrm(Kd) + abs(p.lam) * nrm(Cd) + abs(p.lam) ** 2 * nrm(Md)) * np.linalg.norm(p.u)
        assert np.linalg.norm(r) / den <= 1e-10


def test_real_shift_through_complex_path_matches_real_path():
    P = _perturbed()
    a = rq.solve_quadratic_complex(P, -0.5, 8, m=30, max_restarts=300)
    b = rq.build_operator(P, -0.5).solve_quadratic(8, m=30, eps=1e-10, max_restarts=400)
    la = np.array([p.lam for p in a])
    lb = np.array([p.lam for p in b])
    for x in la:
        assert np.min(np.abs(lb - x)) <= 1e-8 * abs(x)


def test_conductive_maxwell_closed_form():
    """Uniform conductivity sigma = 2 on H(curl) p = 4, 16^2: every eigenvalue
    is i sigma / 2 +- sqrt(kappa - sigma^2 / 4) for a generalized eigenvalue
    kappa of (curl-curl, M); shift at the predicted value for the pair of
    kappa nearest 200 (pi^2 (2^2 + 4^2), double); gyroscopic symmetry."""
    import scipy.sparse.linalg as sla
    P = rq.assemble(rq.CURL, 4, 16, 0)
    sigma = 2.0
    A = P.K - P.M  # curl-curl
    kap = sla.eigsh((P.to_scipy("K") - P.to_scipy("M")).tocsc(), k=4, M=P.to_scipy("M").tocsc(), sigma=200.0,
                    return_eigenvectors=False, tol=1e-13)
    kap = np.sort(kap)
    pred = np.concatenate([1j * sigma / 2 + np.sqrt(kap - sigma ** 2 / 4),
                           1j * sigma / 2 - np.sqrt(kap - sigma ** 2 / 4)])
    s = 1j * sigma / 2 + np.sqrt(kap[2] - sigma ** 2 / 4) + 0.05
    pairs = rq.solve_quadratic_complex(P, s, 2, m=20, eps=1e-10, max_restarts=300,
                                       K=-A, C=-1j * sigma * P.M, M=P.M)
    lam = np.array([p.lam for p in pairs])
    assert max(p.residual for p in pairs) <= 1e-10
    for x in lam:
        assert np.min(np.abs(pred - x)) <= 1e-8 * abs(x)
        assert np.min(np.abs(pred + np.conj(x))) <= 1e-8 * abs(x)  # -conj(lam) is an eigenvalue too


def test_layered_conductive_em_vs_dense_qz_and_symmetry():
    """The paper's conductive EM pencil with two conductivity layers (assemble_em):
    the complex solver's eigenvalues nearest a complex shift equal dense QZ's,
    and the spectrum is symmetric under lam -> -conj(lam) (solving
    at -conj(s) returns the mirrored values)."""
    from scipy.linalg import eigvals
    P = rq.assemble_em(4, 8, layers=((0.0, 0.5, 1.0, 3.0), (0.5, 1.0, 0.2, 0.2)))
    s = 9.0 + 0.8j
    pairs = rq.solve_quadratic_complex(P, s, 4, m=24, eps=1e-10, max_restarts=300)
    lam = np.array([p.lam for p in pairs])
    assert max(p.residual for p in pairs) <= 1e-10
    n = P.n
    Kd, Cd, Md = (P.to_scipy(w).toarray() for w in "KCM")
    Z, I = np.zeros((n, n)), np.eye(n)
    w = eigvals(np.block([[Z, I], [-Kd, -Cd]]), np.block([[I, Z], [Z, Md]]))
    w = w[np.isfinite(w)]
    w = w[np.argsort(np.abs(w - s))][:4]
    for x in lam:
        assert np.min(np.abs(w - x)) <= 1e-8 * abs(x)
    mirror = rq.solve_quadratic_complex(P, -np.conj(s), 4, m=24, eps=1e-10, max_restarts=300)
    lm = np.array([p.lam for p in mirror])
    for x in lam:
        assert np.min(np.abs(lm + np.conj(x))) <= 1e-8 * abs(x)
