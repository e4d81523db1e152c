"""The paper's vibroacoustic quadratic eigenproblem (§6.2.2,
§6.4.2; SPEC.md:225-232 assemble_acoustic, :468 solve_quadratic example;
SURVEY.md §8 row f4 "the paper's acoustic operators") on the B200 path.

Unit-square cavity, rigid walls, one absorbing wall (top), air rho = 1,
c = 340, impedance alpha = 5e4, beta = 200 (Fig. 8). Known answers: the
dispersion equations of PAPER.md:975-990 (eta^2 = lam^2/c^2 + (j pi)^2,
eta tanh(eta) = -rho lam^2 / (alpha + lam beta)) give the purely real
eigenvalues lam_j on the second branch, lam_10 = -7377.39 rad/s quoted by the
paper (reproduced here by root finding); the first branch accumulates at
-alpha/beta = -250 and the branches are separated by -2 alpha/beta = -500;
acoustic stability Re(lam) <= 0.
"""
import numpy as np
import pytest

import oracle
import paper_2112_14064_b200 as rq

pytestmark = pytest.mark.gpu

RHO, C, ALPHA, BETA = 1.0, 340.0, 5e4, 200.0


def dispersion_root(j, lo, hi):
    from scipy.optimize import brentq

    def f(lam):
        eta = np.sqrt(lam ** 2 / C ** 2 + (np.pi * j) ** 2)
        return eta * np.tanh(eta) + RHO * lam ** 2 / (ALPHA + lam * BETA)
    return brentq(f, lo, hi)


def test_acoustic_second_branch_vs_dispersion():
    """p = 3, 32^2 elements, shift -7377: the three nearest eigenvalues are the
    purely real second-branch values of j = 9, 10, 11 (discretisation error
    < 1e-4 relative), pencil residuals <= 1e-10 with scale_pencil on (the
    norms of K and M differ by rho c^2)."""
    P = rq.assemble_acoustic(3, 32)
    op = rq.build_operator(P, -7377.0, scaling=True)
    pairs = op.solve_quadratic(3, m=24, eps=1e-10, max_restarts=400)
    lam = np.array(sorted((p.lam for p in pairs), key=lambda z: z.real))
    assert max(p.residual for p in pairs) <= 1e-10
    assert np.all(np.abs(lam.imag) <= 1e-8 * np.abs(lam))
    exact = np.array(sorted([dispersion_root(j, lo, hi) for j, lo, hi in
                             ((9, -6800.0, -6400.0), (10, -7600.0, -7200.0), (11, -8400.0, -7900.0))]))
    np.testing.assert_allclose(lam.real, exact, rtol=1e-4)


def test_acoustic_branches_near_minus_300():
    """p = 3, ne = 32, nev = 30, shift near -300: purely real
    eigenvalues in two branches separated by -2 alpha / beta = -500 (first
    branch in (-500, -250), accumulating at -alpha / beta), all stable."""
    P = rq.assemble_acoustic(3, 32)
    op = rq.build_operator(P, -300.0, scaling=True)
    pairs = op.solve_quadratic(30, eps=1e-10, max_restarts=400)
    lam = np.array([p.lam for p in pairs])
    assert max(p.residual for p in pairs) <= 1e-10
    assert np.all(np.abs(lam.imag) <= 1e-8 * np.abs(lam))
    assert np.all(lam.real <= 1e-8 * np.abs(lam))
    first = (lam.real > -500.0) & (lam.real < -250.0)
    assert np.all(first | (lam.real < -500.0))
    assert first.sum() >= 20


def test_acoustic_pencil_vs_oracle():
    """GPU eigenvalues of the acoustic pencil (p = 3, 8^2) against the oracle's
    complex Krylov-Schur, both with scale_pencil."""
    P = rq.assemble_acoustic(3, 8)
    op = rq.build_operator(P, -300.0, scaling=True)
    pairs = op.solve_quadratic(8, eps=1e-10, max_restarts=400)
    lam = np.array([p.lam for p in pairs])
    E = oracle.Eig(P, -300.0, scaling=True)
    lo, ro = E.solve_quadratic(8, tol=1e-10, max_restarts=400)
    assert np.all(ro <= 1e-10)
    key = lambda z: (round(abs(z + 300.0), 6), round(z.real, 6))  # noqa: E731
    a = np.array(sorted(lam, key=key))
    b = np.array(sorted(lo, key=key))
    assert np.max(np.abs(a - b) / np.abs(b)) <= 1e-8
