"""GPU parity at the large BASELINE configs (cfg3, cfg4, cfg5) and on a
non-degenerate spectrum, through the C-ABI, against the CPU oracle on the same
seeded inputs.

The oracle's multifrontal LU is tree- and row-parallel over the host cores
(OpenMP, bit-identical for any thread count), so whole cfg4 factorizations
(F_LU 1.8e11 / 6.3e11 real flops, complex arithmetic) finish in tens of seconds
on the GPU box's host and every large front (nf >= 1024, the tiled DMMA path)
is compared entry by entry.

Tolerances (BASELINE north star): pivot sequences bit-exact; L\\U entries
componentwise within 1e-10 of the LU backward-error scale (|L||U|)_ij (same
pivots; summation order differs; see compare_fronts) and within 1e-8 of the
front's largest entry; solves: normwise backward error <= 1e-14; eigenvalues relative 1e-8;
pencil residuals <= 1e-10.
"""
import numpy as np
import pytest

import oracle
import paper_2112_14064_b200 as rq

pytestmark = pytest.mark.gpu

SIGMA = -0.5
CLUSTER = -0.03 + 1j * np.sqrt(0.9991)  # closed form of the degenerate pair


def oracle_kind():
    return "reference" if oracle.ref() is not None else "port"


def all_threads(kind):
    oracle.lib_for(kind).oracle_set_threads(0)


def key(z):
    return (round(abs(z - SIGMA), 7), -np.sign(z.imag), round(z.real, 7))


def sorted_lams(lams):
    return np.array(sorted(lams, key=key))


def backward_error(P, x, b):
    A = P.to_scipy("K") + SIGMA * P.to_scipy("C") + SIGMA ** 2 * P.to_scipy("M")
    nA = abs(A).sum(0).max()
    return np.linalg.norm(A @ x - b, 1) / (nA * np.linalg.norm(x, 1) + np.linalg.norm(b, 1))


def compare_fronts(f, of, o, fronts):
    """Pivot sequences bit-exact, and the L and U panels entry by entry against
    the oracle's, relative to the componentwise backward-error scale of LU with
    those pivots: |dU_ij| <= tau max((|L||U|)_ij, s_f) and
    |dL_ij| |u_jj| <= tau max((|L||U|)_ij, s_f), s_f = 1e-4 max (|L||U|)
    (Higham, Thm 9.3: the computed factors of two summation orders both satisfy
    |A - LU| <= gamma_n |L||U|). A plain max-entry normalisation is not a bound
    here: Q(sigma) = 0.995 div.div + 1.22 M has a large near-kernel, so late
    pivots are ~1e-6 of the front's largest entry and the multipliers they
    divide carry O(n eps / 1e-6) differences. Returns (componentwise,
    max-entry-normalised) worst cases."""
    worst_cw, worst_max = 0.0, 0.0
    for fr in fronts:
        nf, npv = int(o.nf[fr]), int(o.npiv[fr])
        if npv == 0:
            continue
        F, ipiv, _ = f.front(fr)
        Fo, ipo, rows = of.front(fr, nf, npv)
        assert np.array_equal(rows, o.front_rows(fr)), f"front {fr}: row lists differ"
        assert np.array_equal(ipiv, ipo), f"front {fr} (nf {nf}, npiv {npv}): pivots differ"
        G = np.ascontiguousarray(F[:nf, :nf])
        Fo = np.ascontiguousarray(Fo.real)
        La = np.tril(np.abs(Fo[:, :npv]), -1)
        La[np.arange(npv), np.arange(npv)] = 1.0
        Ua = np.triu(np.abs(Fo[:npv, :]))
        S_l = La @ Ua[:, :npv]          # (|L||U|) over the L panel (all rows, pivot columns)
        S_u = La[:npv] @ Ua             # over the U panel (pivot rows, all columns)
        udiag = np.abs(np.diag(Fo[:npv, :npv]))
        dl = np.tril(np.abs(G[:, :npv] - Fo[:, :npv]), -1) * udiag[None, :]
        du = np.triu(np.abs(G[:npv, :] - Fo[:npv, :]))
        tiny = 1e-300
        # floor: entries whose |L||U| scale is below 1e-4 of the front's are
        # exact zeros (explicit fill of the dense ND fronts) in one summation
        # order and roundoff noise in the other; they are held to 1e-4 * tau of
        # the front's scale instead
        floor = 1e-4 * max(np.max(S_l), np.max(S_u))
        worst_cw = max(worst_cw, np.max(dl / np.maximum(S_l, floor)), np.max(du / np.maximum(S_u, floor)))
        d = max(np.max(np.abs(G[:, :npv] - Fo[:, :npv])), np.max(np.abs(G[:npv, :] - Fo[:npv, :])))
        scale = max(np.max(np.abs(Fo[:, :npv])), np.max(np.abs(Fo[:npv, :])), tiny)
        worst_max = max(worst_max, d / scale)
    return worst_cw, worst_max


CW_TOL = 1e-10  # componentwise; observed <= 2.4e-11 (cfg4, cfg5 p = 4, 5 rIGA): ~40 n eps at nf = 2,449


# --------------------------------------------------------------------------- cfg3
@pytest.mark.parametrize("name", ["cfg3_riga", "cfg3_iga"])
def test_cfg3_factor_solve_vs_oracle(name):
    """Every front of the cfg3 factorization (H(curl) p=4 128^2; IGA max front
    1,359 takes the tiled large-front path) against the oracle."""
    P = rq.baseline_config(name)
    o = rq.nested_dissection_order(P)
    Q = P.q_values(SIGMA)
    f = rq.lu_factorize((P.rowptr, P.col, Q), o)
    kind = oracle_kind()
    all_threads(kind)
    of = oracle.Factor(P.n, P.rowptr, P.col, Q, P.box, P.elems, kind=kind)
    assert f.info()["swaps"] == of.swaps
    cw, mx = compare_fronts(f, of, o, range(len(o.nf)))
    assert cw <= CW_TOL and mx <= 1e-8, (cw, mx)
    b = np.random.default_rng(3).standard_normal((P.n, 2))
    x = f.solve(b)
    xo = np.stack([of.solve(b[:, i]).real for i in range(2)], 1)
    assert np.max(np.abs(x - xo)) <= 1e-9 * np.max(np.abs(xo))
    assert backward_error(P, x[:, 0], b[:, 0]) <= 1e-14


@pytest.mark.parametrize("name", ["cfg3_riga", "cfg3_iga"])
def test_cfg3_eigs_vs_oracle(name):
    """BASELINE configs[2] at its own nev = 50 (m = 101): residuals and the
    closed-form cluster value; eigenvalues against the oracle's complex
    Krylov-Schur at nev = 10 (m = 21), the oracle's run at nev = 50 being
    minutes of host time."""
    P = rq.baseline_config(name)
    op = rq.build_operator(P, SIGMA)
    pairs = op.solve_quadratic(50, eps=1e-10, max_restarts=400)
    lam = np.array([p.lam for p in pairs])
    assert len(pairs) == 50 and max(p.residual for p in pairs) <= 1e-10
    assert np.all(np.minimum(np.abs(lam - CLUSTER), np.abs(lam - np.conj(CLUSTER))) <= 1e-8 * abs(CLUSTER))
    pairs10 = op.solve_quadratic(10, eps=1e-10, max_restarts=400)
    lam10 = np.array([p.lam for p in pairs10])
    kind = oracle_kind()
    all_threads(kind)
    E = oracle.Eig(P, SIGMA, kind=kind)
    lo, ro = E.solve_quadratic(10, tol=1e-10, max_restarts=400)
    assert np.max(ro) <= 1e-10
    assert np.max(np.abs(sorted_lams(lam10) - sorted_lams(lo)) / np.abs(lo)) <= 1e-8


# --------------------------------------------------------------------------- cfg4
@pytest.mark.parametrize("name", ["cfg4_riga", "cfg4_iga"])
def test_cfg4_factor_vs_oracle(name):
    """BASELINE configs[3] (H(div) p=3 512^2, N = 0.53-0.59M): one whole
    oracle factorization on the host cores; every front with nf >= 1024 (the
    large-front DMMA path: 55 rIGA / 207 IGA fronts, up to nf 2,449 / 3,846)
    plus every 61st front compared; solve against the oracle and its backward
    error."""
    P = rq.baseline_config(name)
    o = rq.nested_dissection_order(P)
    Q = P.q_values(SIGMA)
    f = rq.lu_factorize((P.rowptr, P.col, Q), o)
    kind = oracle_kind()
    all_threads(kind)
    of = oracle.Factor(P.n, P.rowptr, P.col, Q, P.box, P.elems, kind=kind)
    assert f.info()["swaps"] == of.swaps
    nf = np.asarray(o.nf)
    fronts = sorted(set(np.flatnonzero(nf >= 1024).tolist()) | set(range(0, len(nf), 61)) | {len(nf) - 1})
    cw, mx = compare_fronts(f, of, o, fronts)
    assert cw <= CW_TOL and mx <= 1e-8, (cw, mx)
    b = np.random.default_rng(4).standard_normal(P.n)
    x = f.solve(b)
    xo = of.solve(b).real
    # Q(sigma) at h = 1/512 is ill-conditioned (|x| ~ 3e7 |b|): two backward-
    # stable solves agree to ~cond * eps, so the forward check is 1e-7 relative
    # (observed 1.6e-9) and the backward error carries the 1e-14 bound
    assert np.max(np.abs(x - xo)) <= 1e-7 * np.max(np.abs(xo))
    assert backward_error(P, x, b) <= 1e-14


@pytest.mark.parametrize("name", ["cfg4_riga", "cfg4_iga"])
def test_cfg4_eigs_residuals(name):
    """nev = 100, m = 201 (BASELINE configs[3]): every returned pair converged
    to the explicit pencil residual 1e-10, the cluster value, and a sample of
    residuals recomputed on the host from the returned eigenvectors."""
    P = rq.baseline_config(name)
    op = rq.build_operator(P, SIGMA)
    pairs = op.solve_quadratic(100, eps=1e-10, max_restarts=400, vectors=True)
    assert len(pairs) == 100
    lam = np.array([p.lam for p in pairs])
    assert max(p.residual for p in pairs) <= 1e-10
    assert np.all(np.minimum(np.abs(lam - CLUSTER), np.abs(lam - np.conj(CLUSTER))) <= 1e-8 * abs(CLUSTER))
    K, C, M = (P.to_scipy(w) for w in "KCM")
    nrm = lambda A: abs(A).sum(0).max()  # noqa: E731
    nK, nC, nM = nrm(K), nrm(C), nrm(M)
    for p in pairs[::25]:
        u = p.u
        r = K @ u + p.lam * (C @ u) + p.lam ** 2 * (M @ u)
        assert np.linalg.norm(r) / ((nK + abs(p.lam) * nC + abs(p.lam) ** 2 * nM) * np.linalg.norm(u)) <= 1e-10
    info = op.last_info
    assert info["n_fa"] == 1


@pytest.mark.parametrize("name", ["cfg4_riga", "cfg4_iga"])
def test_cfg4_block_eigs_and_multi_rhs(name):
    """The block path at BASELINE configs[3]: the multi-RHS
    sweeps agree with the single-vector sweeps (8 right-hand sides, relative
    1e-12) and have a backward error <= 1e-14; block Krylov-Schur (block 4)
    returns 100 pairs of the cluster with pencil residuals <= 1e-10, also
    recomputed on the host from the returned vectors."""
    P = rq.baseline_config(name)
    op = rq.build_operator(P, SIGMA)
    f = rq.lu_factorize((P.rowptr, P.col, P.q_values(SIGMA)), op.ordering)
    B = np.random.default_rng(9).standard_normal((P.n, 8))
    x1 = f.solve(B, block=1)
    x8 = f.solve(B, block=8)
    assert np.max(np.abs(x8 - x1)) <= 1e-12 * np.max(np.abs(x1))
    Q = P.to_scipy("K") + SIGMA * P.to_scipy("C") + SIGMA ** 2 * P.to_scipy("M")
    nQ = abs(Q).sum(0).max()
    for j in range(8):
        r = Q @ x8[:, j] - B[:, j]
        assert np.linalg.norm(r, np.inf) / (nQ * np.linalg.norm(x8[:, j], np.inf) + np.linalg.norm(B[:, j], np.inf)) <= 1e-14
    del f
    pairs = op.solve_quadratic(100, eps=1e-10, max_restarts=400, vectors=True, block=4)
    lam = np.array([p.lam for p in pairs])
    assert max(p.residual for p in pairs) <= 1e-10
    assert np.all(np.minimum(np.abs(lam - CLUSTER), np.abs(lam - np.conj(CLUSTER))) <= 1e-8 * abs(CLUSTER))
    K, C, M = (P.to_scipy(w) for w in "KCM")
    nrm = lambda A: abs(A).sum(0).max()  # noqa: E731
    for p in pairs[::25]:
        r = K @ p.u + p.lam * (C @ p.u) + p.lam ** 2 * (M @ p.u)
        den = (nrm(K) + abs(p.lam) * nrm(C) + abs(p.lam) ** 2 * nrm(M)) * np.linalg.norm(p.u)
        assert np.linalg.norm(r) / den <= 1e-10
    assert op.last_info["restart_defect"] <= 1e-10


# --------------------------------------------------------------------------- cfg5
@pytest.mark.parametrize("p", [2, 3, 4, 5])
@pytest.mark.parametrize("disc", ["iga", "riga"])
def test_cfg5_factor_backward_error(p, disc):
    """BASELINE configs[4] part 1 (H(curl) 256^2, p = 2..5, IGA vs rIGA):
    factorization + solve backward error; against a whole oracle factorization
    (rIGA trees and IGA p <= 3: the IGA p = 4, 5 trees cost minutes of host
    time) the 8 largest fronts and every 97th front."""
    name = f"cfg5_p{p}_{disc}"
    P = rq.baseline_config(name)
    o = rq.nested_dissection_order(P)
    Q = P.q_values(SIGMA)
    f = rq.lu_factorize((P.rowptr, P.col, Q), o)
    b = np.random.default_rng(p).standard_normal(P.n)
    x = f.solve(b)
    assert backward_error(P, x, b) <= 1e-14
    if disc == "riga" or p <= 3:
        kind = oracle_kind()
        all_threads(kind)
        of = oracle.Factor(P.n, P.rowptr, P.col, Q, P.box, P.elems, kind=kind)
        nf = np.asarray(o.nf)
        fronts = sorted(set(np.argsort(nf)[-8:].tolist()) | set(range(0, len(nf), 97)))
        cw, mx = compare_fronts(f, of, o, fronts)
        assert cw <= CW_TOL and mx <= 1e-8, (cw, mx)


# --------------------------------------------------------------------------- spectrum
def test_nondegenerate_spectrum_cfg2_riga_vs_oracle():
    """The BASELINE pencils' requested pairs are copies of one degenerate
    eigenvalue, so eigenvalue parity on them is nearly vacuous. Here cfg2 rIGA's
    damping gets a random positive diagonal (C += 0.5 u_i M_ii, u ~ U[0,1)):
    the 20 eigenvalues nearest the shift are distinct, and both solvers must
    find the same ones."""
    P = rq.baseline_config("cfg2_riga")
    diag = np.array([P.rowptr[i] + np.searchsorted(P.col[P.rowptr[i]:P.rowptr[i + 1]], i) for i in range(P.n)])
    rng = np.random.default_rng(2024)
    P.C = P.C.copy()
    P.C[diag] += 0.5 * rng.random(P.n) * P.M[diag]
    op = rq.build_operator(P, SIGMA)
    pairs = op.solve_quadratic(20, eps=1e-10, max_restarts=400)
    lam = sorted_lams([p.lam for p in pairs])
    assert max(p.residual for p in pairs) <= 1e-10
    # distinct: no two requested values within 1e-6 relative
    gaps = np.abs(lam[:, None] - lam[None, :]) + np.eye(len(lam))
    assert gaps.min() > 1e-6
    kind = oracle_kind()
    all_threads(kind)
    E = oracle.Eig(P, SIGMA, kind=kind, C_=P.C)
    lo, ro = E.solve_quadratic(20, tol=1e-10, max_restarts=400)
    assert np.max(ro) <= 1e-10
    assert np.max(np.abs(lam - sorted_lams(lo)) / np.abs(lo)) <= 1e-8


@pytest.mark.parametrize("name", ["cfg3_riga", "cfg3_iga"])
def test_streamed_refactor_matches_resident_factor(name):
    """rq_factor_refactor uploads the values in chunks while the task-DAG kernel
    runs (tasks wait for their own entries; FactorEngine::factor_streamed): the
    factors must be those of a factorization with the values resident (the
    first factorization of a handle, and lu_factorize on the new values)."""
    P = rq.baseline_config(name)
    assert P.nnz >= 1 << 20  # below that the refactor uploads first
    o = rq.nested_dissection_order(P)
    Q = P.q_values(-0.5)
    b = np.random.default_rng(7).uniform(-1.0, 1.0, P.n)
    f = rq.lu_factorize((P.rowptr, P.col, Q), o)  # values resident
    x0 = f.solve(b)
    for _ in range(3):
        f.refactor(Q)  # streamed
        assert np.array_equal(f.solve(b), x0)
    Q2 = P.q_values(-0.7)
    f.refactor(Q2)  # streamed, new values
    x2 = f.solve(b)
    g = rq.lu_factorize((P.rowptr, P.col, Q2), o)
    assert np.array_equal(g.solve(b), x2)
    import scipy.sparse as sp
    A = sp.csr_matrix((Q2, P.col, P.rowptr), shape=(P.n, P.n))
    nA = abs(A).sum(0).max()
    assert np.linalg.norm(A @ x2 - b, 1) / (nA * np.linalg.norm(x2, 1) + np.linalg.norm(b, 1)) <= 1e-14


def test_streamed_refactor_concurrent_handles():
    """Two threads refactor their own handles from host values at the same time
    (two persistent factor kernels, each waiting for its own streamed chunks):
    both must finish and reproduce the serial results bit for bit."""
    import threading

    jobs = []
    for name in ("cfg3_riga", "cfg3_iga"):
        P = rq.baseline_config(name)
        o = rq.nested_dissection_order(P)
        Q = P.q_values(-0.5)
        b = np.random.default_rng(11).uniform(-1.0, 1.0, P.n)
        f = rq.lu_factorize((P.rowptr, P.col, Q), o)
        jobs.append({"f": f, "Q": Q, "b": b, "x0": f.solve(b), "out": [], "err": None})

    def work(j):
        try:
            for _ in range(6):
                j["f"].refactor(j["Q"])
                j["out"].append(j["f"].solve(j["b"]))
        except Exception as e:  # noqa: BLE001
            j["err"] = e

    ts = [threading.Thread(target=work, args=(j,)) for j in jobs]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in ts), "concurrent streamed refactors did not finish"
    for j in jobs:
        assert j["err"] is None, j["err"]
        assert len(j["out"]) == 6
        for x in j["out"]:
            assert np.array_equal(x, j["x0"])
