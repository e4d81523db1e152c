"""Host-side SPEC operations of the eig module through the C-ABI (no GPU):
scale_pencil and ritz_extract, with the
SPEC's own examples and a dense-eigensolver oracle."""
import numpy as np
import pytest

import paper_2112_14064_b200 as rq


class _P:
    def __init__(self, K, C, M):
        self.K, self.C, self.M = (np.asarray(a, float) for a in (K, C, M))


def test_scale_pencil_known_answers():
    # K = 4I, C = M = I -> varsigma = 2, scaled pencil (4I, 2I, 4I)
    vs, Cs, Ms = rq.scale_pencil(_P(4 * np.ones(3), np.ones(3), np.ones(3)))
    assert vs == 2.0 and np.array_equal(Cs, 2 * np.ones(3)) and np.array_equal(Ms, 4 * np.ones(3))
    # equal norms -> varsigma = 1, pencil unchanged
    vs, Cs, Ms = rq.scale_pencil(_P([1.0, -2.0], [3.0, 5.0], [2.0, 1.0]))
    assert vs == 1.0 and np.array_equal(Cs, [3.0, 5.0]) and np.array_equal(Ms, [2.0, 1.0])
    # zero M -> domain error
    with pytest.raises(rq.RqError) as e:
        rq.scale_pencil(_P([1.0], [1.0], [0.0]))
    assert e.value.category == "domain"


def test_scale_pencil_matches_oracle(cfg1):
    import oracle
    vs, Cs, Ms = rq.scale_pencil(cfg1)
    vo, Co, Mo = oracle.scale_pencil(cfg1.n, cfg1.rowptr, cfg1.col, cfg1.K, cfg1.C, cfg1.M)
    assert vs == vo and np.array_equal(Cs, Co.real) and np.array_equal(Ms, Mo.real)


def hess(m, beta, rng):
    H = np.zeros((m + 1, m))
    H[:m] = np.triu(rng.standard_normal((m, m)), -1)
    H[m, m - 1] = beta
    return H


def test_ritz_extract_spec_examples():
    # H = diag(2, 3), s = 0 -> lambda = 1/2, 1/3
    H = np.array([[2.0, 0.0], [0.0, 3.0], [0.0, 0.0]])
    r = rq.ritz_extract(H, 0.0)
    assert np.allclose(sorted(r["lambda"].real), [1 / 3, 1 / 2], rtol=1e-15)
    assert np.all(r["est"] == 0.0)
    # [[0, 1], [1, 0]] -> theta = +-1
    r = rq.ritz_extract(np.array([[0.0, 1.0], [1.0, 0.0], [0.0, 0.0]]), 0.0)
    assert np.allclose(sorted(r["theta"].real), [-1.0, 1.0], atol=1e-15)


@pytest.mark.parametrize("m", [8, 21, 60])
def test_ritz_extract_vs_dense(m):
    """eigenvalues of a random Hessenberg vs a dense oracle to 1e-9;
    wanted order; Ritz vectors, residual estimates and the back-transform."""
    rng = np.random.default_rng(m)
    H = hess(m, 0.37, rng)
    sigma, vs = -0.5, 1.7
    r = rq.ritz_extract(H, sigma, vs)
    Hm = H[:m]
    w = np.linalg.eigvals(Hm)
    for t in r["theta"]:
        assert np.min(np.abs(w - t)) <= 1e-9 * max(1.0, abs(t))
    assert np.allclose(r["lambda"], sigma + vs / r["theta"], rtol=1e-14)
    d = np.abs(r["lambda"] - sigma)
    assert np.all(np.diff(d) >= -1e-12 * d[1:])  # nearest the shift first
    Y = r["y"]
    assert np.allclose(np.linalg.norm(Y, axis=0), 1.0, atol=1e-12)
    assert np.max(np.abs(Hm @ Y - Y * r["theta"][None, :])) <= 1e-9 * np.abs(Hm).max()
    assert np.allclose(r["est"], np.abs(0.37 * Y[m - 1]), rtol=1e-12, atol=1e-300)


def test_ritz_extract_dimension_errors():
    with pytest.raises(rq.RqError) as e:
        rq.ritz_extract(np.zeros((3, 3)), 0.0)
    assert e.value.category == "dimension"
