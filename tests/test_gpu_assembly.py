"""Device assembly of the BASELINE pencil vs the host
assembler (csrc/host/spaces.cpp:assemble_pencil).

The device path must reproduce the host pencil bit for bit: pattern (integer)
and K, C, M (every product and sum rounded separately on both sides, element
contributions summed in the host's colour order)."""
import numpy as np
import pytest

import paper_2112_14064_b200 as rq

pytestmark = pytest.mark.gpu


def _same(P, Q):
    assert P.n == Q.n and P.n_full == Q.n_full
    assert np.array_equal(P.rowptr, Q.rowptr)
    assert np.array_equal(P.col, Q.col)
    assert np.array_equal(P.box, Q.box)
    assert np.array_equal(P.free_to_full, Q.free_to_full)
    for a, b in ((P.K, Q.K), (P.C, Q.C), (P.M, Q.M)):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("args", [
    (rq.DIV, 2, 8, 0), (rq.CURL, 2, 8, 2), (rq.DIV, 3, 64, 3), (rq.CURL, 4, 32, 2),
    (rq.CURL, 5, 64, 3), (rq.DIV, 7, 16, 1),
    (rq.CURL, 12, 6, 0),   # shared-memory chunking of the Gauss points (rows < nq)
])
def test_device_assembly_bitexact(args):
    ms = np.zeros(5)
    H = rq.assemble(*args)
    D = rq.assemble(*args, device=True, stage_ms=ms)
    _same(H, D)
    assert np.all(ms[:3] > 0)


def test_device_assembly_damping_coefficients():
    H = rq.assemble(rq.DIV, 3, 16, 1, alpha=0.3, beta=0.07)
    D = rq.assemble(rq.DIV, 3, 16, 1, alpha=0.3, beta=0.07, device=True)
    _same(H, D)


@pytest.mark.parametrize("name", ["cfg2_riga", "cfg3_iga"])
def test_device_assembly_baseline_configs(name):
    _same(rq.baseline_config(name), rq.baseline_config(name, device=True))


def test_device_assembled_pencil_eigensolve():
    """The device-assembled pencil feeds the eigensolver directly (same pairs)."""
    P = rq.baseline_config("cfg1", device=True)
    op = rq.build_operator(P, -0.5)
    pairs = op.solve_quadratic(6, eps=1e-10, seed=0)
    assert len(pairs) >= 6
    assert max(p.residual for p in pairs[:6]) <= 1e-10


def test_resident_pencil_values_on_demand():
    H = rq.baseline_config("cfg2_riga")
    D = rq.baseline_config("cfg2_riga", device=True, resident=True)
    assert getattr(D, "device_resident", False)
    _same(H, D)   # K, C, M copied out of HBM on first access


@pytest.mark.parametrize("scaling", [False, True])
@pytest.mark.parametrize("name", ["cfg1", "cfg2_riga"])
def test_resident_operator_equals_host_operator(name, scaling):
    """Operator built in place from the device-assembled pencil (Q(s), scaling
    and residual norms formed on the device) gives the host operator's results
    bit for bit."""
    H = rq.baseline_config(name)
    D = rq.baseline_config(name, device=True, resident=True)
    oh = rq.build_operator(H, -0.5, scaling=scaling)
    od = rq.build_operator(D, -0.5, scaling=scaling)
    assert oh.varsigma == od.varsigma
    fh, fd = oh.factor_info(), od.factor_info()
    assert fh["swaps"] == fd["swaps"]
    x = np.random.default_rng(3).standard_normal(H.n)
    for w in "KCMQ":
        assert np.array_equal(oh.spmv(w, x), od.spmv(w, x))
    v = np.random.default_rng(4).standard_normal(2 * H.n)
    assert np.array_equal(oh.apply(v), od.apply(v))
    ph = oh.solve_quadratic(8, eps=1e-10, seed=0)
    pd = od.solve_quadratic(8, eps=1e-10, seed=0)
    assert [p.lam for p in ph] == [p.lam for p in pd]
    assert [p.residual for p in ph] == [p.residual for p in pd]


def test_device_pencil_export_matches_host_export(tmp_path):
    """f3 pencil export straight from a device-resident pencil (one copy out of
    HBM) writes the same bytes as the host pencil's export."""
    H = rq.baseline_config("cfg1")
    D = rq.baseline_config("cfg1", device=True, resident=True)
    fh = rq.write_pencil(H, str(tmp_path / "h_"))
    fd = rq.write_pencil(D, str(tmp_path / "d_"))
    for a, b in zip(fh, fd):
        assert open(a, "rb").read() == open(b, "rb").read()
