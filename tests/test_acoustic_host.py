"""Host side of the paper's vibroacoustic problem (
SPEC.md:225-232 assemble_acoustic): the dispersion known answer and the
structure of the assembled pencil (no GPU needed)."""
import numpy as np

import paper_2112_14064_b200 as rq

RHO, C, ALPHA, BETA = 1.0, 340.0, 5e4, 200.0


def test_dispersion_known_answer():
    """The paper's lam_10 = -7377.39 rad/s from the dispersion
    equations on the unit square (second branch, lam < -2 alpha / beta)."""
    from scipy.optimize import brentq

    def f(lam, j=10):
        eta = np.sqrt(lam ** 2 / C ** 2 + (np.pi * j) ** 2)
        return eta * np.tanh(eta) + RHO * lam ** 2 / (ALPHA + lam * BETA)
    assert abs(brentq(f, -7600.0, -7200.0) - (-7377.39)) <= 0.005


def test_acoustic_pencil_structure():
    """C only on the absorbing wall's normal DOFs (the top wall: y-component,
    last basis row), K, C, M symmetric, K = rho c^2 div-div + alpha term, M =
    rho mass; no absorbing wall -> C = 0 and the rigid BASELINE mask; the edge
    mass integrates the constant to the wall length (sum of C / beta = 1)."""
    P = rq.assemble_acoustic(3, 8)
    Cd = P.to_scipy("C")
    rows = np.unique(Cd.nonzero()[0])
    top_y = set(range(P.n_full - (3 + 8 - 1), P.n_full))
    assert set(P.free_to_full[rows].tolist()) <= top_y and len(rows) == 3 + 8 - 1
    for w in "KCM":
        A = P.to_scipy(w)
        assert abs(A - A.T).max() == 0.0
    # partition of unity of the tangential space: sum_ij int B_i B_j = |wall| = 1
    assert abs(Cd.sum() / BETA - 1.0) <= 1e-13
    P0 = rq.assemble_acoustic(3, 8, absorbing=())
    assert np.abs(P0.C).max() == 0.0
    B = rq.assemble(rq.DIV, 3, 8, 0)
    assert P0.n == B.n and np.array_equal(P0.col, B.col)
    np.testing.assert_allclose(P0.M, RHO * B.M, rtol=0, atol=1e-15 * np.abs(B.M).max())
    np.testing.assert_allclose(P0.K, RHO * C * C * (B.K - B.M), rtol=0, atol=1e-12 * np.abs(P0.K).max())


def test_em_pencil_structure():
    """assemble_em: K = -(1/mu) curl-curl, M = eps mass, C = -i D;
    uniform conductivity -> D = sigma M; layered: D only weights the layers' rows
    (sigma 0 above 0.5 -> D smaller than the uniform one), symmetric."""
    B = rq.assemble(rq.CURL, 4, 8, 0)
    P = rq.assemble_em(4, 8, mu=2.0, eps=3.0, layers=((0.0, 1.0, 2.0, 2.0),))
    assert np.iscomplexobj(P.C) and np.all(P.C.real == 0)
    np.testing.assert_allclose(P.K, -(B.K - B.M) / 2.0, rtol=0, atol=1e-14 * np.abs(B.K).max())
    np.testing.assert_allclose(P.M, 3.0 * B.M, rtol=0, atol=1e-15 * np.abs(B.M).max())
    np.testing.assert_allclose(-P.C.imag, 2.0 * B.M, rtol=0, atol=1e-14 * np.abs(B.M).max())
    L = rq.assemble_em(4, 8, layers=((0.0, 0.5, 1.0, 3.0), (0.5, 1.0, 0.0, 0.0)))
    Dd = -np.asarray(L.to_scipy("C").toarray()).imag
    assert np.abs(Dd - Dd.T).max() <= 1e-15 * np.abs(Dd).max()
    assert Dd.trace() < (3.0 * B.to_scipy("M")).diagonal().sum()
