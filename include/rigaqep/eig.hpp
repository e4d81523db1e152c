// SPDX-License-Identifier: Apache-2.0
// eig drop-in for the reference tree, over the B200 C-ABI
// (include/rq_b200.h). Real pencils and real shifts only on the GPU path
// (errc::config otherwise; no CPU fallback). Complex vectors are applied as
// two real applications and charged as the one operation the reference
// performs. Every CostLedger charge is read back from the operator's own
// ledger (rq_operator_ledger), which follows the reference operations one for
// one.
#pragma once

#include <algorithm>
#include <complex>
#include <cstring>
#include <memory>
#include <vector>

#include "rigaqep/sparsela.hpp"

namespace rq {

/// QuadraticPencil: K, C, M on one shared pattern. The
/// ordering is the pencil's symbolic analysis (make_pencil attaches the
/// geometric nested dissection of its space); without one, solve_quadratic
/// uses the natural ordering (one dense front: small pencils only).
struct QuadraticPencil {
  SparseMatrix K, C, M;
  std::shared_ptr<const Ordering> ordering;
  double varsigma = 1.0;  // scaling state: 1 = unscaled
  long N() const { return K.n; }
};

inline QuadraticPencil make_pencil(const VectorSpace& vs, const std::vector<long>& constrained, SparseMatrix K,
                                   SparseMatrix C, SparseMatrix M) {
  QuadraticPencil p{std::move(K), std::move(C), std::move(M), nullptr};
  p.ordering = std::make_shared<Ordering>(nested_dissection_order(vs, constrained));
  if (p.ordering->n() != p.N()) fail(errc::dimension, "make_pencil: space and matrices differ in size");
  return p;
}

struct EigenPair {
  cdouble lambda;
  std::vector<cdouble> u;  // unit 2-norm, larger-norm block of the Ritz vector
  double residual = 0.0;
};

/// ShiftInvertOperator: device-resident factor of Q(s).
struct ShiftInvertOperator {
  std::shared_ptr<rq_operator_t> op;
  cdouble s;
  long n = 0;
  double varsigma = 1.0;
};

namespace b200 {
inline void same_pattern(const QuadraticPencil& p) {
  if (p.C.rowptr != p.K.rowptr || p.M.rowptr != p.K.rowptr || p.C.col != p.K.col || p.M.col != p.K.col)
    fail(errc::dimension, "K, C, M must share one pattern (SPEC.md:263)");
}
inline void ledger_snapshot(const ShiftInvertOperator& op, double* out) {
  check(rq_operator_ledger(op.op.get(), out));
}
/// charge the reference CostLedger with the operator-ledger delta after - before
/// (ops and multiply-adds per category); `scale_ops` = 1 / number of real
/// applications a complex operation took
inline void charge(CostLedger* L, const double* before, const double* after, int real_parts = 1) {
  if (!L) return;
  void (CostLedger::*add[6])(std::uint64_t) = {&CostLedger::add_fa, &CostLedger::add_fb, &CostLedger::add_mv,
                                               &CostLedger::add_vv, &CostLedger::add_check, &CostLedger::add_restart};
  for (int c = 0; c < 6; ++c) {
    const auto ops = static_cast<std::uint64_t>((after[2 * c] - before[2 * c]) / real_parts);
    const auto macs = static_cast<std::uint64_t>((after[2 * c + 1] - before[2 * c + 1]) / real_parts);
    for (std::uint64_t k = 0; k < ops; ++k) (L->*add[c])(k == 0 ? macs : 0);
  }
}
inline bool is_real(const std::vector<cdouble>& v) {
  return std::all_of(v.begin(), v.end(), [](const cdouble& z) { return z.imag() == 0.0; });
}
}  // namespace b200

/// scale_pencil: returns (K, varsigma C, varsigma^2 M) and
/// varsigma = sqrt(maxabs K / maxabs M); zero M -> errc::domain.
inline std::pair<QuadraticPencil, double> scale_pencil(const QuadraticPencil& p) {
  b200::same_pattern(p);
  const std::vector<double> K = real_values(p.K), C = real_values(p.C), M = real_values(p.M);
  std::vector<double> Cs(C.size()), Ms(M.size());
  double vs = 1.0;
  b200::check(rq_scale_pencil(static_cast<std::int64_t>(K.size()), K.data(), C.data(), M.data(), &vs, Cs.data(),
                              Ms.data()));
  QuadraticPencil q = p;
  for (std::size_t k = 0; k < Cs.size(); ++k) q.C.val[k] = Cs[k], q.M.val[k] = Ms[k];
  q.varsigma = p.varsigma * vs;
  return {std::move(q), vs};
}

/// build_operator: one LU factorization of Q(s), N_fa = 1.
inline ShiftInvertOperator build_operator(const QuadraticPencil& p, cdouble s, const Ordering& ord,
                                          CostLedger* ledger, bool scaling = false) {
  if (s.imag() != 0.0) fail(errc::config, "the B200 path takes real shifts only");
  b200::same_pattern(p);
  if (ord.n() != p.N()) fail(errc::dimension, "build_operator: ordering and pencil sizes differ");
  const std::vector<double> K = real_values(p.K), C = real_values(p.C), M = real_values(p.M);
  rq_operator_opts o{s.real(), scaling ? 1 : 0};
  rq_operator_t* h = nullptr;
  b200::check(rq_operator_create(p.N(), p.K.rowptr.data(), p.K.col.data(), K.data(), C.data(), M.data(),
                                 ord.sym.get(), &o, &h));
  ShiftInvertOperator op;
  op.op.reset(h, rq_operator_destroy);
  op.s = s;
  op.n = p.N();
  op.varsigma = rq_operator_varsigma(h);
  double z[12] = {0}, a[12];
  b200::ledger_snapshot(op, a);
  b200::charge(ledger, z, a);
  return op;
}

/// apply_operator: r_u = -Q(s)^{-1}(s M v_u + C v_u + M v_l),
/// r_l = s r_u + v_u on v = (v_u; v_l). Charges 1 fb, 3 mv, 3 vv.
inline std::vector<cdouble> apply_operator(const ShiftInvertOperator& op, const std::vector<cdouble>& v,
                                           CostLedger* ledger) {
  const long n2 = 2 * op.n;
  if (static_cast<long>(v.size()) != n2) fail(errc::dimension, "apply_operator dimension mismatch");
  const bool real = b200::is_real(v);
  std::vector<double> a(n2), b(n2), ra(n2), rb(n2, 0.0);
  for (long i = 0; i < n2; ++i) a[i] = v[i].real(), b[i] = v[i].imag();
  double l0[12], l1[12];
  b200::ledger_snapshot(op, l0);
  b200::check(rq_operator_apply(op.op.get(), a.data(), ra.data()));
  if (!real) b200::check(rq_operator_apply(op.op.get(), b.data(), rb.data()));
  b200::ledger_snapshot(op, l1);
  b200::charge(ledger, l0, l1, real ? 1 : 2);
  std::vector<cdouble> r(n2);
  for (long i = 0; i < n2; ++i) r[i] = {ra[i], rb[i]};
  return r;
}

/// b_inner: x_u^H y_u + x_l^H M y_l (one B-product, one dot).
inline cdouble b_inner(const ShiftInvertOperator& op, const std::vector<cdouble>& x, const std::vector<cdouble>& y,
                       CostLedger* ledger) {
  const long n2 = 2 * op.n;
  if (static_cast<long>(x.size()) != n2 || static_cast<long>(y.size()) != n2)
    fail(errc::dimension, "b_inner dimension mismatch");
  std::vector<double> xr(n2), xi(n2), yr(n2), yi(n2);
  for (long i = 0; i < n2; ++i) xr[i] = x[i].real(), xi[i] = x[i].imag(), yr[i] = y[i].real(), yi[i] = y[i].imag();
  const bool real = b200::is_real(x) && b200::is_real(y);
  double l0[12], l1[12];
  b200::ledger_snapshot(op, l0);
  double rr = 0, ii = 0, ri = 0, ir = 0;  // x^H y = (xr - i xi)(yr + i yi)
  b200::check(rq_operator_b_inner(op.op.get(), xr.data(), yr.data(), &rr));
  b200::ledger_snapshot(op, l1);
  if (!real) {
    b200::check(rq_operator_b_inner(op.op.get(), xi.data(), yi.data(), &ii));
    b200::check(rq_operator_b_inner(op.op.get(), xr.data(), yi.data(), &ri));
    b200::check(rq_operator_b_inner(op.op.get(), xi.data(), yr.data(), &ir));
  }
  b200::charge(ledger, l0, l1);
  return {rr + ii, ri - ir};
}

/// KrylovState: V (m+1 vectors of 2N, upper; lower halves),
/// H (m+1) x m column-major, beta = h_{m+1,m}, Nit = Arnoldi steps run.
struct KrylovState {
  std::vector<std::vector<cdouble>> V;
  std::vector<cdouble> H;
  int m = 0;
  double beta = 0.0;
  long nit = 0;
  cdouble h(int i, int j) const { return H[i + static_cast<std::size_t>(j) * (m + 1)]; }
};

/// arnoldi_run: m-step B-orthogonal Arnoldi with CGS2 from
/// v1 (B-normalised first); M is the operator's mass matrix (B = diag(I, M)).
inline KrylovState arnoldi_run(const ShiftInvertOperator& op, const SparseMatrix& M, int m,
                               const std::vector<cdouble>& v1, CostLedger* ledger) {
  const long n2 = 2 * op.n;
  if (M.n != op.n) fail(errc::dimension, "arnoldi_run: M does not match the operator");
  if (static_cast<long>(v1.size()) != n2) fail(errc::dimension, "arnoldi_run: v1 dimension mismatch");
  if (!b200::is_real(v1)) fail(errc::config, "the B200 path runs real Krylov spaces (real v1)");
  if (m < 1 || m >= n2) fail(errc::config, "arnoldi_run: m must be in [1, 2N)");
  std::vector<double> v(n2), V(static_cast<std::size_t>(m + 1) * n2), H(static_cast<std::size_t>(m + 1) * m);
  for (long i = 0; i < n2; ++i) v[i] = v1[i].real();
  double l0[12], l1[12];
  b200::ledger_snapshot(op, l0);
  b200::check(rq_operator_arnoldi(op.op.get(), v.data(), m, V.data(), H.data()));
  b200::ledger_snapshot(op, l1);
  b200::charge(ledger, l0, l1);
  KrylovState S;
  S.m = m;
  S.nit = m;
  S.V.assign(m + 1, std::vector<cdouble>(n2));
  for (int j = 0; j <= m; ++j)
    for (long i = 0; i < n2; ++i) S.V[j][i] = V[static_cast<std::size_t>(j) * n2 + i];
  S.H.assign(H.begin(), H.end());
  S.beta = H[m + static_cast<std::size_t>(m - 1) * (m + 1)];
  return S;
}

/// ritz_extract: one entry per Ritz value, wanted order.
struct RitzValue {
  cdouble theta, lambda;
  std::vector<cdouble> y;  // in the H basis, unit 2-norm
  double residual_estimate = 0.0;  // |beta e_m^H y|
};

inline std::vector<RitzValue> ritz_extract(const KrylovState& state, const ShiftInvertOperator& op) {
  const int m = state.m;
  std::vector<double> H(static_cast<std::size_t>(m + 1) * m);
  for (std::size_t k = 0; k < H.size(); ++k) {
    if (state.H[k].imag() != 0.0) fail(errc::config, "the B200 path extracts from real Hessenberg matrices");
    H[k] = state.H[k].real();
  }
  std::vector<double> th(2 * m), lam(2 * m), est(m), Y(2 * static_cast<std::size_t>(m) * m);
  b200::check(rq_ritz_extract(H.data(), m, op.s.real(), op.varsigma, th.data(), lam.data(), est.data(), Y.data()));
  std::vector<RitzValue> out(m);
  for (int a = 0; a < m; ++a) {
    out[a].theta = {th[2 * a], th[2 * a + 1]};
    out[a].lambda = {lam[2 * a], lam[2 * a + 1]};
    out[a].residual_estimate = est[a];
    out[a].y.resize(m);
    for (int r = 0; r < m; ++r)
      out[a].y[r] = {Y[2 * (r + static_cast<std::size_t>(a) * m)], Y[2 * (r + static_cast<std::size_t>(a) * m) + 1]};
  }
  return out;
}

/// krylov_schur_restart: keep the `keep` wanted directions
/// (conjugate pairs kept whole); `nev` is the caller's target (keep >= nev).
inline KrylovState krylov_schur_restart(const ShiftInvertOperator& op, const KrylovState& state, int nev, int keep,
                                        CostLedger* ledger) {
  if (keep < nev) fail(errc::config, "krylov_schur_restart: keep must be at least nev");
  const int m = state.m;
  const long n2 = 2 * op.n;
  std::vector<double> V(static_cast<std::size_t>(m + 1) * n2), H(static_cast<std::size_t>(m + 1) * m);
  for (int j = 0; j <= m; ++j)
    for (long i = 0; i < n2; ++i) V[static_cast<std::size_t>(j) * n2 + i] = state.V[j][i].real();
  for (std::size_t k = 0; k < H.size(); ++k) H[k] = state.H[k].real();
  int p = 0;
  double l0[12], l1[12];
  b200::ledger_snapshot(op, l0);
  b200::check(rq_operator_krylov_schur_restart(op.op.get(), m, keep, V.data(), H.data(), &p));
  b200::ledger_snapshot(op, l1);
  b200::charge(ledger, l0, l1);
  KrylovState S;
  S.m = p;
  S.nit = state.nit;
  S.V.assign(p + 1, std::vector<cdouble>(n2));
  for (int j = 0; j <= p; ++j)
    for (long i = 0; i < n2; ++i) S.V[j][i] = V[static_cast<std::size_t>(j) * n2 + i];
  S.H.assign(static_cast<std::size_t>(p + 1) * p, 0.0);
  for (int c = 0; c < p; ++c)
    for (int i = 0; i <= p; ++i) S.H[i + static_cast<std::size_t>(c) * (p + 1)] = H[i + static_cast<std::size_t>(c) * (m + 1)];
  S.beta = 0.0;
  return S;
}

/// solve_quadratic: nev pairs nearest s with relative pencil
/// residual <= eps; m > nev (m <= 0 selects 2 nev + 1, BASELINE). Fails with
/// errc::solver (partial result) after max_restarts.
inline std::vector<EigenPair> solve_quadratic(const QuadraticPencil& p, cdouble s, int nev, int m, double eps,
                                              CostLedger* ledger, std::uint64_t seed = 0, int max_restarts = 100) {
  const Ordering ord = p.ordering ? *p.ordering : natural_order(p.N());
  const ShiftInvertOperator op = build_operator(p, s, ord, ledger);
  rq_eigs_opts o{nev, m, eps, seed, max_restarts, 1, 0, 1};
  std::vector<double> lr(nev), li(nev), res(nev), vr(static_cast<std::size_t>(op.n) * nev),
      vi(static_cast<std::size_t>(op.n) * nev);
  rq_eigs_info info{};
  double l0[12], l1[12];
  b200::ledger_snapshot(op, l0);
  const int rc = rq_eigs_run(op.op.get(), &o, lr.data(), li.data(), res.data(), vr.data(), vi.data(), &info);
  b200::ledger_snapshot(op, l1);
  b200::charge(ledger, l0, l1);
  b200::check(rc);
  std::vector<EigenPair> out(nev);
  for (int i = 0; i < nev; ++i) {
    out[i].lambda = {lr[i], li[i]};
    out[i].residual = res[i];
    out[i].u.resize(op.n);
    for (long k = 0; k < op.n; ++k) out[i].u[k] = {vr[i * op.n + k], vi[i * op.n + k]};
  }
  return out;
}

}  // namespace rq
