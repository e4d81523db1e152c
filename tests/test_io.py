"""Wire formats: Matrix Market files and the eigenpair
JSON dump, pinned byte for byte against the reference's own writers / reader
(sparse.cpp:121-174, compiled into oracle/_ref) and cross-checked with scipy."""
import json
import os

import numpy as np
import pytest
import scipy.io
import scipy.sparse as sp

import paper_2112_14064_b200 as rq
from oracle import ref_mm

needs_ref = pytest.mark.skipif(not ref_mm.available(), reason="reference sources not built here (oracle/_ref)")


def _bytes(path):
    return open(path, "rb").read()


@pytest.fixture(scope="module")
def cfg1():
    return rq.baseline_config("cfg1")


@needs_ref
@pytest.mark.parametrize("which", ["K", "C", "M"])
def test_pencil_matrix_bytes_equal_reference_writer(cfg1, which, tmp_path):
    mine, theirs = str(tmp_path / "mine.mtx"), str(tmp_path / "ref.mtx")
    vals = getattr(cfg1, which)
    rq.write_matrix_market((cfg1.rowptr, cfg1.col, vals), mine)
    ref_mm.write(cfg1.rowptr, cfg1.col, vals, None, theirs)
    assert _bytes(mine) == _bytes(theirs)


@needs_ref
def test_complex_matrix_and_special_values_bytes_equal(tmp_path):
    rng = np.random.default_rng(5)
    A = sp.random(40, 40, density=0.2, random_state=7, format="csr")
    A.sort_indices()
    re = rng.standard_normal(A.nnz) * 10.0 ** rng.integers(-300, 300, A.nnz)
    im = rng.standard_normal(A.nnz)
    re[:4] = [0.0, -0.0, 1.0 / 3.0, 2.0 ** -1074]
    im[:3] = [0.0, -0.0, 1e308]
    mine, theirs = str(tmp_path / "mine.mtx"), str(tmp_path / "ref.mtx")
    val = np.empty(A.nnz, complex)
    val.real, val.imag = re, im   # (re + 1j * im would turn an imaginary -0.0 into +0.0)
    rq.write_matrix_market((A.indptr, A.indices, val), mine)
    ref_mm.write(A.indptr, A.indices, re, im, theirs)
    assert _bytes(mine) == _bytes(theirs)
    assert _bytes(mine).startswith(b"%%MatrixMarket matrix coordinate complex general\n40 40 ")


@needs_ref
def test_vector_bytes_equal_reference_writer(tmp_path):
    x = np.random.default_rng(1).standard_normal(257) + 1j * np.random.default_rng(2).standard_normal(257)
    mine, theirs = str(tmp_path / "mine.mtx"), str(tmp_path / "ref.mtx")
    rq.write_matrix_market_vector(x, mine)
    ref_mm.write_vector(x.real, x.imag, theirs)
    assert _bytes(mine) == _bytes(theirs)


@needs_ref
def test_read_sums_duplicates_like_reference(tmp_path):
    path = str(tmp_path / "dup.mtx")
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate complex general\n% a comment\n4 4 7\n"
                "3 1 1.5 0\n1 1 2 1\n3 1 0.25 -1\n4 4 -1 0\n2 3 7 0\n1 1 -0.5 0.5\n4 2 0 0\n")
    rowptr, col, val = rq.read_matrix_market(path)
    rp, cl, re, im = ref_mm.read(path)
    assert np.array_equal(rowptr, rp) and np.array_equal(col, cl)
    assert np.array_equal(val.real, re) and np.array_equal(val.imag, im)
    assert val[0] == 1.5 + 1.5j and len(cl) == 5   # (1,1) summed; explicit zero kept


def test_roundtrip_and_scipy_crosscheck(cfg1, tmp_path):
    prefix = str(tmp_path / "cfg1_")
    files = rq.write_pencil(cfg1, prefix)
    for w, path in zip("KCM", files):
        rowptr, col, val = rq.read_matrix_market(path)
        assert np.array_equal(rowptr, cfg1.rowptr) and np.array_equal(col, cfg1.col)
        assert np.array_equal(val, getattr(cfg1, w))          # %.17g round-trips doubles exactly
        S = scipy.io.mmread(path).tocsr()
        assert (abs(S - cfg1.to_scipy(w))).max() == 0.0


def test_vector_scipy_crosscheck(tmp_path):
    x = np.linspace(-1, 1, 33) * (1 + 0.5j)
    path = str(tmp_path / "v.mtx")
    rq.write_matrix_market_vector(x, path)
    y = scipy.io.mmread(path).ravel()
    assert np.array_equal(x, y)


def test_eigenpair_json_dump(tmp_path):
    pairs = [rq.EigenPair(complex(-0.03, 0.9995), 3.2e-11), rq.EigenPair(complex(-1.0 / 3.0, -0.0), 0.0)]
    s = rq.eigenpairs_json(pairs)
    d = json.loads(s)
    assert [(e["re"], e["im"], e["residual"]) for e in d] == [(-0.03, 0.9995, 3.2e-11), (-1.0 / 3.0, -0.0, 0.0)]
    path = str(tmp_path / "pairs.json")
    rq.write_eigenpairs(pairs, path)
    assert rq.load_eigenpairs(path) == [(p.lam, p.residual) for p in pairs]
    assert rq.eigenpairs_json([]) == "[]"


def test_errors(tmp_path):
    with pytest.raises(rq.RqError):
        rq.read_matrix_market(str(tmp_path / "missing.mtx"))
    bad = tmp_path / "bad.mtx"
    bad.write_text("not a matrix\n")
    with pytest.raises(rq.RqError):
        rq.read_matrix_market(str(bad))
    trunc = tmp_path / "trunc.mtx"
    trunc.write_text("%%MatrixMarket matrix coordinate real general\n3 3 4\n1 1 1.0\n")
    with pytest.raises(rq.RqError):
        rq.read_matrix_market(str(trunc))
    with pytest.raises(rq.RqError):
        rq.write_matrix_market((np.array([0, 0]), np.array([], np.int32), np.array([])),
                               str(tmp_path / "no_such_dir" / "x.mtx"))
