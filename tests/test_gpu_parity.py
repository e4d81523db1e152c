"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle on the
same seeded inputs, plus size-independent properties at larger sizes.

Tolerances (floating point, BASELINE north star): eigenvalues relative 1e-8,
pencil residuals <= 1e-10; factor entries / solves relative 1e-10 against the
oracle (both are backward-stable FP64 LU with the same pivot sequence; the
difference is summation order, bounded by cond(A) * eps); integer work (pivot
sequences, orderings) bit-exact.
"""
import numpy as np
import pytest

import oracle
import paper_2112_14064_b200 as rq

pytestmark = pytest.mark.gpu

SIGMA = -0.5


def key(z):
    return (round(abs(z - SIGMA), 7), -np.sign(z.imag), round(z.real, 7))


def sorted_lams(lams):
    return np.array(sorted(lams, key=key))


class Tiny:
    def __init__(self, A):
        A = np.asarray(A, float)
        n = A.shape[0]
        self.n, self.elems = n, 1
        self.rowptr = np.arange(0, n * n + 1, n, dtype=np.int64)
        self.col = np.tile(np.arange(n, dtype=np.int32), n)
        self.val = A.ravel()
        self.box = np.zeros((n, 4), np.int32)


def dense_factor(A):
    t = Tiny(A)
    o = rq.Ordering(t.n, t.box, 1)
    return rq.lu_factorize((t.rowptr, t.col, t.val), o), o


# --------------------------------------------------------------------------- factor
def test_lu_known_answer_3x3():
    A = [[4, 3, 0], [6, 3, 1], [0, 1, 2]]
    f, o = dense_factor(A)
    F, ipiv, ld = f.front(0)
    assert list(ipiv) == [0, 1, 2] and f.info()["swaps"] == 0
    np.testing.assert_allclose(np.tril(F[:3, :3], -1), [[0, 0, 0], [1.5, 0, 0], [0, -2 / 3, 0]], atol=1e-15)
    np.testing.assert_allclose(np.triu(F[:3, :3]), [[4, 3, 0], [0, -1.5, 1], [0, 0, 8 / 3]], atol=1e-15)
    np.testing.assert_allclose(np.asarray(A) @ f.solve(np.array([1.0, 2, 3])), [1, 2, 3], atol=1e-14)


def test_identity_and_spd50():
    f, _ = dense_factor(np.eye(5))
    x = np.arange(5.0)
    np.testing.assert_array_equal(f.solve(x), x)
    rng = np.random.default_rng(0)
    B = rng.standard_normal((50, 50))
    A = B @ B.T + 50 * np.eye(50)
    f, _ = dense_factor(A)
    b = rng.standard_normal(50)
    assert np.linalg.norm(A @ f.solve(b) - b) / np.linalg.norm(b) <= 1e-12


@pytest.mark.parametrize("n", [40, 170, 700, 1500])
def test_dense_pivoting_matches_oracle(n):
    """Single front through the SMEM (n<=160) and blocked/cluster (n>160) paths:
    pivot sequence bit-exact, L\\U entries vs the oracle."""
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n))
    A[np.arange(n), np.arange(n)] *= 0.05  # force threshold swaps
    f, _ = dense_factor(A)
    F, ipiv, ld = f.front(0)
    t = Tiny(A)
    of = oracle.Factor(n, t.rowptr, t.col, t.val, t.box, 1)
    Fo, ipo, _ = of.front(0, n, n)
    assert np.array_equal(ipiv, ipo)
    assert f.info()["swaps"] == of.swaps > 0
    err = np.max(np.abs(F[:n, :n] - Fo.real)) / np.max(np.abs(Fo))
    assert err <= 1e-13 * n  # same pivots; summation order differs (growth ~ n eps)
    b = rng.standard_normal(n)
    x = f.solve(b)
    assert np.linalg.norm(A @ x - b) <= 1e-11 * np.linalg.norm(A, 1) * np.linalg.norm(x)


def test_singular_is_reported():
    A = np.ones((4, 4))
    with pytest.raises(rq.RqError) as e:
        dense_factor(A)
    assert e.value.category == "singular"


@pytest.mark.parametrize("name,sched", [("cfg1", "dag"), ("cfg2_riga", "dag"), ("cfg2_iga", "dag"),
                                        ("cfg2_riga", "level")])
def test_multifrontal_vs_oracle(name, sched, monkeypatch):
    """Default task-DAG schedule, and the level-synchronous A/B path (RQB_FACTOR=level)."""
    if sched == "level":
        monkeypatch.setenv("RQB_FACTOR", "level")
    P = rq.baseline_config(name)
    o = rq.nested_dissection_order(P)
    Q = P.q_values(SIGMA)
    f = rq.lu_factorize((P.rowptr, P.col, Q), o)
    of = oracle.Factor(P.n, P.rowptr, P.col, Q, P.box, P.elems)
    # every front: pivots bit-exact, factor entries within 1e-10 relative
    worst = 0.0
    for fr in range(0, len(o.nf), max(1, len(o.nf) // 40)):
        nf, npv = int(o.nf[fr]), int(o.npiv[fr])
        F, ipiv, _ = f.front(fr)
        Fo, ipo, rows = of.front(fr, nf, npv)
        assert np.array_equal(rows, o.front_rows(fr))
        assert np.array_equal(ipiv, ipo)
        # compare the factor part (L and U panels)
        mask = np.zeros((nf, nf), bool)
        mask[:, :npv] = True
        mask[:npv, :] = True
        d = np.max(np.abs((F[:nf, :nf] - Fo.real)[mask])) / max(np.max(np.abs(Fo.real[mask])), 1e-300)
        worst = max(worst, d)
    assert worst <= 1e-10
    rng = np.random.default_rng(7)
    b = rng.standard_normal((P.n, 3))
    x = f.solve(b)
    xo = np.stack([of.solve(b[:, i]).real for i in range(3)], 1)
    assert np.max(np.abs(x - xo)) <= 1e-9 * np.max(np.abs(xo))
    A = P.to_scipy("K") + SIGMA * P.to_scipy("C") + SIGMA ** 2 * P.to_scipy("M")
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) <= 1e-10


def test_refactor_same_pattern(cfg1):
    o = rq.nested_dissection_order(cfg1)
    f = rq.lu_factorize((cfg1.rowptr, cfg1.col, cfg1.q_values(SIGMA)), o)
    Q2 = cfg1.q_values(-1.5)
    f.refactor(Q2)
    A = cfg1.to_scipy("K") - 1.5 * cfg1.to_scipy("C") + 2.25 * cfg1.to_scipy("M")
    b = np.ones(cfg1.n)
    assert np.linalg.norm(A @ f.solve(b) - b) / np.linalg.norm(b) <= 1e-10


# --------------------------------------------------------------------------- operator
@pytest.mark.parametrize("name", ["cfg1", "cfg2_riga"])
def test_apply_spmv_binner_vs_oracle(name):
    P = rq.baseline_config(name)
    op = rq.build_operator(P, SIGMA)
    E = oracle.Eig(P, SIGMA)
    rng = np.random.default_rng(3)
    v = rng.uniform(-1, 1, 2 * P.n)
    r = op.apply(v)
    ro = E.apply(v).real
    assert np.max(np.abs(r - ro)) <= 1e-9 * np.max(np.abs(ro))
    x = rng.standard_normal(P.n)
    for w in "KCM":
        y = op.spmv(w, x)
        ys = P.to_scipy(w) @ x
        assert np.max(np.abs(y - ys)) <= 1e-13 * np.max(np.abs(ys))
    y = rng.standard_normal(2 * P.n)
    bi = op.b_inner(v, y)
    ref = v[:P.n] @ y[:P.n] + v[P.n:] @ (P.to_scipy("M") @ y[P.n:])
    assert abs(bi - ref) <= 1e-12 * abs(ref) + 1e-14


def test_arnoldi_invariants(cfg1):
    """Arnoldi identity and B-orthonormality <= 1e-8."""
    op = rq.build_operator(cfg1, SIGMA)
    n = cfg1.n
    v1 = np.random.default_rng(0).uniform(-1, 1, 2 * n)
    m = 21
    V, H = op.arnoldi(v1, m)
    Mm = cfg1.to_scipy("M")
    BV = np.concatenate([V[:, :n], (Mm @ V[:, n:].T).T], 1)
    G = V @ BV.T
    assert np.max(np.abs(G - np.eye(m + 1))) <= 1e-8
    SV = np.stack([op.apply(V[j]) for j in range(m)])
    R = SV.T - V.T @ H
    assert np.max(np.abs(R)) <= 1e-8 * np.max(np.abs(H))
    assert np.allclose(np.tril(H, -2), 0)


# --------------------------------------------------------------------------- eigensolve
def test_eigs_cfg1_vs_oracle(cfg1):
    op = rq.build_operator(cfg1, SIGMA)
    pairs = op.solve_quadratic(10, eps=1e-10, seed=0, vectors=True)
    lam = np.array([p.lam for p in pairs])
    res = np.array([p.residual for p in pairs])
    E = oracle.Eig(cfg1, SIGMA)
    lo, ro = E.solve_quadratic(10, tol=1e-10, seed=0)
    a, b = sorted_lams(lam), sorted_lams(lo)
    assert np.max(np.abs(a - b) / np.abs(b)) <= 1e-8
    assert np.all(res <= 1e-10)
    ref = -0.03 + 1j * np.sqrt(0.9991)  # closed form of the degenerate cluster
    assert np.all(np.minimum(np.abs(lam - ref), np.abs(lam - np.conj(ref))) <= 1e-8 * abs(ref))
    # eigenvector residual recomputed on the host
    K, C, M = (cfg1.to_scipy(w) for w in "KCM")
    for p in pairs[:4]:
        u = p.u
        r = K @ u + p.lam * (C @ u) + p.lam ** 2 * (M @ u)
        nrm = lambda A: abs(A).sum(0).max()  # noqa: E731
        den = (nrm(K) + abs(p.lam) * nrm(C) + abs(p.lam) ** 2 * nrm(M)) * np.linalg.norm(u)
        assert np.linalg.norm(r) / den <= 1e-10
    info = op.last_info
    assert info["n_fa"] == 1 and info["restart_defect"] <= 1e-10
    # counter laws: one solve per Arnoldi step, 4..6 mv per step
    assert 4 <= info["n_mv"] / info["n_fb"] <= 7


def test_eigs_nondegenerate_vs_oracle_and_scipy():
    """Perturbed damping breaks the cluster: parity of a generic spectrum."""
    from scipy.linalg import eigvals
    P = rq.assemble(rq.DIV, 2, 8, 0)
    diag = np.array([P.rowptr[i] + np.searchsorted(P.col[P.rowptr[i]:P.rowptr[i + 1]], i)
                     for i in range(P.n)])
    rng = np.random.default_rng(11)
    P.C = P.C.copy()
    P.C[diag] += 0.5 * rng.random(P.n) * P.M[diag]
    op = rq.build_operator(P, SIGMA)
    pairs = op.solve_quadratic(8, eps=1e-10, max_restarts=400)
    lam = np.array([p.lam for p in pairs])
    E = oracle.Eig(P, SIGMA, C_=P.C)
    lo, _ = E.solve_quadratic(8, tol=1e-10, max_restarts=400)
    assert np.max(np.abs(sorted_lams(lam) - sorted_lams(lo)) / np.abs(lo)) <= 1e-8
    n = P.n
    Kd, Cd, Md = (P.to_scipy(w).toarray() for w in "KCM")
    Z, I = np.zeros((n, n)), np.eye(n)
    w = eigvals(np.block([[Z, I], [-Kd, -Cd]]), np.block([[I, Z], [Z, Md]]))
    w = w[np.argsort(np.abs(w - SIGMA))][:8]
    for x in lam:
        assert np.min(np.abs(w - x)) <= 1e-8 * abs(x)


def test_eigs_cfg2_riga_vs_oracle(cfg2r):
    op = rq.build_operator(cfg2r, SIGMA)
    pairs = op.solve_quadratic(20, eps=1e-10, max_restarts=400)
    lam = np.array([p.lam for p in pairs])
    E = oracle.Eig(cfg2r, SIGMA)
    lo, _ = E.solve_quadratic(20, tol=1e-10, max_restarts=400)
    assert np.max(np.abs(sorted_lams(lam) - sorted_lams(lo)) / np.abs(lo)) <= 1e-8
    assert max(p.residual for p in pairs) <= 1e-10


def test_scaling_does_not_change_spectrum(cfg1):
    a = rq.build_operator(cfg1, SIGMA, scaling=False).solve_quadratic(6)
    b = rq.build_operator(cfg1, SIGMA, scaling=True).solve_quadratic(6)
    la, lb = sorted_lams([p.lam for p in a]), sorted_lams([p.lam for p in b])
    assert np.max(np.abs(la - lb) / np.abs(la)) <= 1e-6


def test_scale_pencil_vs_oracle():
    """scale_pencil: the product's varsigma equals the
    oracle's bit for bit, and the scaled solve's eigenvalues match the oracle's
    scaled solve (perturbed damping: a non-degenerate spectrum)."""
    P = rq.assemble(rq.DIV, 2, 8, 0)
    diag = np.array([P.rowptr[i] + np.searchsorted(P.col[P.rowptr[i]:P.rowptr[i + 1]], i) for i in range(P.n)])
    P.C = P.C.copy()
    P.C[diag] += 0.5 * np.random.default_rng(9).random(P.n) * P.M[diag]
    op = rq.build_operator(P, SIGMA, scaling=True)
    vs, Cs, Ms = oracle.scale_pencil(P.n, P.rowptr, P.col, P.K, P.C, P.M)
    assert op.varsigma == vs and vs != 1.0
    assert np.max(np.abs(Ms.real - vs * vs * P.M)) == 0.0
    # nev = 5: one real value and two conjugate pairs (an even count would
    # split a pair, and which member is returned is arbitrary)
    pairs = op.solve_quadratic(5, eps=1e-10, max_restarts=400)
    E = oracle.Eig(P, SIGMA, C_=P.C, scaling=True)
    assert E.varsigma == vs
    lo, ro = E.solve_quadratic(5, tol=1e-10, max_restarts=400)
    lam = sorted_lams([p.lam for p in pairs])
    assert np.max(np.abs(lam - sorted_lams(lo)) / np.abs(lo)) <= 1e-8
    assert max(p.residual for p in pairs) <= 1e-10 and np.max(ro) <= 1e-10


# --------------------------------------------------------------------------- larger sizes
@pytest.mark.parametrize("name", ["cfg3_riga", "cfg3_iga"])
def test_cfg3_solve_residual_and_cluster(name):
    P = rq.baseline_config(name)
    op = rq.build_operator(P, SIGMA)
    fac = rq.lu_factorize((P.rowptr, P.col, P.q_values(SIGMA)), op.ordering)
    A = P.to_scipy("K") + SIGMA * P.to_scipy("C") + SIGMA ** 2 * P.to_scipy("M")
    b = np.random.default_rng(1).standard_normal(P.n)
    x = fac.solve(b)
    # normwise backward error (Q(sigma) is ill-conditioned at this mesh size)
    nA = abs(A).sum(0).max()
    assert np.linalg.norm(A @ x - b, 1) / (nA * np.linalg.norm(x, 1) + np.linalg.norm(b, 1)) <= 1e-14
    pairs = op.solve_quadratic(10, eps=1e-10, max_restarts=400)
    ref = -0.03 + 1j * np.sqrt(0.9991)
    lam = np.array([p.lam for p in pairs])
    assert np.all(np.minimum(np.abs(lam - ref), np.abs(lam - np.conj(ref))) <= 1e-8 * abs(ref))
    assert max(p.residual for p in pairs) <= 1e-10


# --------------------------------------------------------------------------- sweeps
@pytest.mark.parametrize("name", ["cfg1", "cfg2_riga"])
def test_solve_whole_front_items_and_determinism(name, monkeypatch):
    """The triangular sweeps' item layouts (64-row blocks with in-front waits;
    whole small fronts per CTA, enabled by default only on levels with >= 2 x
    grid fronts; backward partial items over contribution-column chunks, forced
    here with 64-column chunks) give the oracle's solution, and
    repeated solves are bitwise identical (per-block partial sums are added in
    block order, independent of publication timing)."""
    P = rq.baseline_config(name)
    o = rq.nested_dissection_order(P)
    Q = P.q_values(SIGMA)
    of = oracle.Factor(P.n, P.rowptr, P.col, Q, P.box, P.elems)
    b = np.random.default_rng(11).standard_normal((P.n, 2))
    xo = np.stack([of.solve(b[:, i]).real for i in range(2)], 1)
    xs = []
    for whole_min, chunk in ((None, None), ("1", None), (None, "64")):
        if whole_min is None:
            monkeypatch.delenv("RQB_WHOLE_MIN", raising=False)
        else:
            monkeypatch.setenv("RQB_WHOLE_MIN", whole_min)
        if chunk is None:  # backward partial items over contribution-column chunks (default: > 256 columns)
            monkeypatch.delenv("RQB_CB_CHUNK", raising=False)
        else:
            monkeypatch.setenv("RQB_CB_CHUNK", chunk)
        f = rq.lu_factorize((P.rowptr, P.col, Q), o)
        x1, x2 = f.solve(b), f.solve(b)
        assert np.array_equal(x1, x2)
        assert np.max(np.abs(x1 - xo)) <= 1e-9 * np.max(np.abs(xo))
        xs.append(x1)
    monkeypatch.delenv("RQB_WHOLE_MIN", raising=False)
    monkeypatch.delenv("RQB_CB_CHUNK", raising=False)
    for x in xs[1:]:
        assert np.max(np.abs(xs[0] - x)) <= 1e-12 * np.max(np.abs(xs[0]))


@pytest.mark.parametrize("name,occ,batch", [("cfg1", "1", None), ("cfg1", "2", None), ("cfg2_riga", "1", None),
                                            ("cfg2_riga", "2", "2"), ("cfg2_riga", "2", "4")])
def test_pivoting_in_every_front_vs_oracle(name, occ, batch, monkeypatch):
    """Threshold pivoting inside a multifrontal tree (the BASELINE pencils never
    swap): cfg1's pattern with random values and a weak diagonal, so most
    fronts swap. Both kernel variants (and the throughput variant's deferred
    UPDB batches of 2 and 4 steps with a 1-step lookahead, so row swaps of the
    fallback meet pending batches): occ 1 (SMALL fronts up to nf 160, the
    exact warp-shuffle panel), occ 2 (SMALL up to 118: the 119..145 fronts take
    the tiled path, whose speculative panel fails and is redone by the exact
    fallback with contribution rows and children present); cfg2 rIGA's fronts
    up to nf 325 take the tiled path in either variant. Pivots bit-exact, factor
    entries and the solution against the oracle."""
    P = rq.baseline_config(name)
    o = rq.nested_dissection_order(P)
    rng = np.random.default_rng(5)
    Q = rng.standard_normal(P.nnz)
    rows = np.repeat(np.arange(P.n), np.diff(P.rowptr))
    Q[P.col == rows] *= 0.01
    monkeypatch.setenv("RQB_DAG_OCC", occ)
    if batch:  # deferred (UPDB) updates with threshold-pivoting fallbacks in flight
        monkeypatch.setenv("RQB_UPD_BATCH", batch)
        monkeypatch.setenv("RQB_UPD_LOOKAHEAD", "1")
    f = rq.lu_factorize((P.rowptr, P.col, Q), o)
    monkeypatch.delenv("RQB_DAG_OCC")
    monkeypatch.delenv("RQB_UPD_BATCH", raising=False)
    monkeypatch.delenv("RQB_UPD_LOOKAHEAD", raising=False)
    of = oracle.Factor(P.n, P.rowptr, P.col, Q, P.box, P.elems)
    assert f.info()["swaps"] == of.swaps > 0
    worst = 0.0
    for fr in range(len(o.nf)):
        nf, npv = int(o.nf[fr]), int(o.npiv[fr])
        F, ipiv, _ = f.front(fr)
        Fo, ipo, _ = of.front(fr, nf, npv)
        assert np.array_equal(ipiv, ipo), f"front {fr} (nf {nf}, npiv {npv})"
        mask = np.zeros((nf, nf), bool)
        mask[:, :npv] = True
        mask[:npv, :] = True
        d = np.max(np.abs((F[:nf, :nf] - Fo.real)[mask])) / max(np.max(np.abs(Fo.real[mask])), 1e-300)
        worst = max(worst, d)
    assert worst <= 1e-9
    b = rng.standard_normal(P.n)
    x = f.solve(b)
    xo = of.solve(b).real
    assert np.max(np.abs(x - xo)) <= 1e-8 * np.max(np.abs(xo))


# --------------------------------------------------------------------------- evidence entry
def test_schur_update_bench_entry():
    """rq_factor_bench_updcb (the factorization's own contribution-block Schur
    update over one front, timed alone) runs on a large-front problem, reports
    the front's update work, and a refactorization afterwards restores a
    factorization that solves to the oracle's accuracy."""
    from paper_2112_14064_b200 import _lib
    P = rq.baseline_config("cfg3_riga")
    o = rq.nested_dissection_order(P)
    Q = P.q_values(SIGMA)
    f = rq.lu_factorize((P.rowptr, P.col, Q), o)
    out = np.zeros(6)
    _lib.check(_lib.lib.rq_factor_bench_updcb(f._h, -1, 2, out))
    front, K = int(out[2]), int(out[4])
    assert out[0] > 0 and out[3] >= 1 and K == o.npiv[front]
    m = o.nf[front] - (o.npiv[front] + 63) // 64 * 64  # rows/columns of the contribution-block tiles
    assert out[1] == pytest.approx(2.0 * K * m * m)
    f.refactor(Q)
    b = np.random.default_rng(5).standard_normal(P.n)
    x = f.solve(b)
    r = P.to_scipy("K") @ x - 0.5 * (P.to_scipy("C") @ x) + 0.25 * (P.to_scipy("M") @ x) - b
    assert np.linalg.norm(r) <= 1e-9 * np.linalg.norm(b)


# --------------------------------------------------------------------------- ledger / SPEC operations
def test_ledger_matches_oracle_per_operation(cfg1):
    """CostLedger parity (sparse.hpp:57-103): build_operator,
    apply_operator, b_inner and arnoldi_run charge exactly the counters the
    reference CPU path (the oracle's rq::spmv / dot / axpy sequence) charges;
    N_vv of arnoldi_run grows quadratically in m."""
    op = rq.build_operator(cfg1, SIGMA)
    E = oracle.Eig(cfg1, SIGMA)
    assert op.ledger_counts() == E.ledger_counts()  # fa: one factorization
    assert op.ledger_counts()["fa"][0] == 1
    rng = np.random.default_rng(1)
    v = rng.uniform(-1, 1, 2 * cfg1.n)
    op.ledger_reset(), E.ledger_reset()
    op.apply(v), E.apply(v)
    assert op.ledger_counts() == E.ledger_counts()
    assert op.ledger_counts()["fb"][0] == 1 and op.ledger_counts()["mv"][0] == 3
    x, y = rng.standard_normal(2 * cfg1.n), rng.standard_normal(2 * cfg1.n)
    op.ledger_reset(), E.ledger_reset()
    bo, bg = E.b_inner(x, y), op.b_inner(x, y)
    assert abs(bo.real - bg) <= 1e-12 * abs(bg)
    assert op.ledger_counts() == E.ledger_counts()
    vv = {}
    for m in (20, 40, 80):
        op.ledger_reset(), E.ledger_reset()
        op.arnoldi(v, m), E.arnoldi(v, m)
        g, o = op.ledger_counts(), E.ledger_counts()
        assert g == o, (m, g, o)
        assert g["fb"][0] == m and g["mv"][0] == 6 * m + 1
        vv[m] = g["vv"][0]
    assert 3.5 <= vv[40] / vv[20] <= 4.0 and 3.5 <= vv[80] / vv[40] <= 4.0  # ~ 2 m^2
    js = op.ledger_json()
    assert set(js) == {"fa", "fb", "mv", "vv", "residual_check", "restart", "flops_per_mac", "total_flops"}


def test_solve_quadratic_counter_laws(cfg1):
    """N_fa = 1 per solve; one operator application (N_fb) per
    Arnoldi step; N_mv / N_fb in [4, 6] plus the start vectors' B-products;
    the operator's cumulative ledger adds the solve's (fa charged once)."""
    op = rq.build_operator(cfg1, SIGMA)
    op.solve_quadratic(10, eps=1e-10)
    info, led = op.last_info, op.ledger
    assert info["n_fa"] == 1 and led["fa"]["ops"] == 1
    assert 6.0 <= info["n_mv"] / info["n_fb"] <= 6.2
    assert info["n_restart"] >= 1 and info["n_check"] >= 10
    cum = op.ledger_counts()
    assert cum["fa"][0] == 1 and cum["fb"][0] == info["n_fb"] and cum["vv"][0] == info["n_vv"]
    # a repeated solve replays the cached cycle graphs: same launch count;
    # after release_workspace the graphs are rebuilt: same again
    op.solve_quadratic(10, eps=1e-10)
    assert op.last_info["launches"] == info["launches"]
    op.release_workspace()
    op.solve_quadratic(10, eps=1e-10)
    assert op.last_info["launches"] == info["launches"]


def test_krylov_schur_restart_invariants(cfg1):
    """after keeping the wanted directions, S V_p = V_p T_p +
    v_{p+1} b^T holds, V_{p+1} stays B-orthonormal, the kept Ritz values are
    the wanted ones of H_m, and keep >= m is the identity restart."""
    op = rq.build_operator(cfg1, SIGMA)
    n, m = cfg1.n, 21
    V, H = op.arnoldi(np.random.default_rng(2).uniform(-1, 1, 2 * n), m)
    r = op.ritz_extract(H)
    Vp, Hp, p = op.krylov_schur_restart(V, H, 11)
    assert 11 <= p <= 12 and Vp.shape == (p + 1, 2 * n) and Hp.shape == (p + 1, p)
    Mm = cfg1.to_scipy("M")
    BV = np.concatenate([Vp[:, :n], (Mm @ Vp[:, n:].T).T], 1)
    assert np.max(np.abs(Vp @ BV.T - np.eye(p + 1))) <= 1e-10
    SV = np.stack([op.apply(Vp[j]) for j in range(p)])
    R = SV.T - Vp.T @ Hp
    assert np.max(np.abs(R)) <= 1e-8 * np.max(np.abs(H))
    kept = np.linalg.eigvals(Hp[:p])
    for t in r["theta"][:p]:
        assert np.min(np.abs(kept - t)) <= 1e-10 * abs(t)
    V2, H2, p2 = op.krylov_schur_restart(V, H, m)
    assert p2 == m and np.array_equal(V2, V) and np.array_equal(H2, H)


def test_tma_bulk_staging_path_matches_oracle(monkeypatch):
    """The opt-in TMA bulk-copy staging of the K-batched Schur updates
    (RQB_UPD_TMA=1, cp.async.bulk + mbarrier) gives the oracle's factors."""
    P = rq.baseline_config("cfg3_iga")
    o = rq.nested_dissection_order(P)
    Q = P.q_values(SIGMA)
    monkeypatch.setenv("RQB_UPD_TMA", "1")
    f = rq.lu_factorize((P.rowptr, P.col, Q), o)
    b = np.random.default_rng(8).standard_normal(P.n)
    x = f.solve(b)
    monkeypatch.delenv("RQB_UPD_TMA")
    g = rq.lu_factorize((P.rowptr, P.col, Q), o)
    x2 = g.solve(b)
    assert np.max(np.abs(x - x2)) <= 1e-9 * np.max(np.abs(x2))
    A = P.to_scipy("K") + SIGMA * P.to_scipy("C") + SIGMA ** 2 * P.to_scipy("M")
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) <= 1e-9


# --------------------------------------------------------------------------- complex LU
@pytest.mark.parametrize("name", ["cfg1", "cfg2_riga"])
def test_complex_shift_factor_solve_vs_oracle(name):
    """Q(s) at a complex shift s = -0.5 + 0.3i (complex-symmetric, SPEC.md:311
    over complex scalars): factored on the GPU as its real-equivalent 2n system
    (rq_factor_create_complex), solved for complex right-hand sides; against
    the oracle's native complex multifrontal LU (the reference's cdouble
    arithmetic) within 1e-9, normwise backward error <= 1e-14, and a real
    right-hand side's solution differs from the real-shift one."""
    import scipy.sparse as sp
    P = rq.baseline_config(name)
    s = -0.5 + 0.3j
    Qv = P.K + s * P.C + s * s * P.M
    o = rq.nested_dissection_order(P)
    f = rq.lu_factorize((P.rowptr, P.col, Qv), o)
    assert f.is_complex
    rng = np.random.default_rng(2)
    b = rng.standard_normal(P.n) + 1j * rng.standard_normal(P.n)
    x = f.solve(b)
    Qs = sp.csr_matrix((Qv, P.col, P.rowptr), shape=(P.n, P.n))
    r = Qs @ x - b
    nQ = abs(Qs).sum(0).max()
    assert np.linalg.norm(r, np.inf) / (nQ * np.linalg.norm(x, np.inf) + np.linalg.norm(b, np.inf)) <= 1e-14
    of = oracle.Factor(P.n, P.rowptr, P.col, Qv, P.box, P.elems)
    xo = of.solve(b)
    assert np.max(np.abs(x - xo)) <= 1e-9 * np.max(np.abs(xo))
    # the real entry points refuse a complex factorization (their buffers are n, not 2n)
    with pytest.raises(rq.RqError) as e:
        rq.sparsela._lib.check(rq.sparsela._lib.lib.rq_factor_solve_ex(f._h, np.zeros(2 * P.n), np.zeros(2 * P.n), 1, 1))
    assert e.value.code == 2
    # several right-hand sides at once (multi-RHS sweeps over the 2n system)
    B = rng.standard_normal((P.n, 3)) + 1j * rng.standard_normal((P.n, 3))
    X = f.solve(B)
    for j in range(3):
        assert np.max(np.abs(X[:, j] - f.solve(B[:, j]))) <= 1e-12 * np.max(np.abs(X[:, j]))
