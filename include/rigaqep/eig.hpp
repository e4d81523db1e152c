// SPDX-License-Identifier: Apache-2.0
// eig drop-in for the reference tree, over the B200 C-ABI.
// Real pencils and real shifts only on the GPU path (errc::config otherwise).
#pragma once

#include <complex>
#include <memory>
#include <vector>

#include "rigaqep/sparsela.hpp"

namespace rq {

/// QuadraticPencil: K, C, M on one shared pattern.
struct QuadraticPencil {
  SparseMatrix K, C, M;
  long N() const { return K.n; }
};

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

inline void same_pattern(const QuadraticPencil& p) {
  if (p.C.rowptr != p.K.rowptr || p.M.rowptr != p.K.rowptr || p.C.col != p.K.col ||
      p.M.col != p.K.col)
    fail(errc::dimension, "K, C, M must share one pattern (SPEC.md:263)");
}

/// build_operator: N_fa = 1.
inline ShiftInvertOperator build_operator(const QuadraticPencil& p, cdouble s, const Ordering& ord,
                                          CostLedger* ledger, bool scaling = false) {
  if (s.imag() != 0.0) fail(errc::config, "the B200 path takes real shifts only");
  same_pattern(p);
  const std::vector<double> K = real_values(p.K), C = real_values(p.C), M = real_values(p.M);
  rq_operator_opts o{s.real(), scaling ? 1 : 0};
  rq_operator_t* h = nullptr;
  b200::check(rq_operator_create(p.N(), p.K.rowptr.data(), p.K.col.data(), K.data(), C.data(),
                                 M.data(), ord.sym.get(), &o, &h));
  ShiftInvertOperator op;
  op.op.reset(h, rq_operator_destroy);
  op.s = s;
  op.n = p.N();
  op.varsigma = rq_operator_varsigma(h);
  if (ledger) {
    rq_symbolic_stats st{};
    b200::check(rq_symbolic_stats_get(ord.sym.get(), &st));
    ledger->add_fa(static_cast<std::uint64_t>(st.flops_lu / 2));
  }
  return op;
}

/// apply_operator on v = (v_u; v_l), complex input split
/// into two real applications.
inline std::vector<cdouble> apply_operator(const ShiftInvertOperator& op, const std::vector<cdouble>& v,
                                           CostLedger* ledger) {
  const long n2 = 2 * op.n;
  if (static_cast<long>(v.size()) != n2) fail(errc::dimension, "apply_operator dimension mismatch");
  std::vector<double> a(n2), b(n2), ra(n2), rb(n2);
  for (long i = 0; i < n2; ++i) a[i] = v[i].real(), b[i] = v[i].imag();
  b200::check(rq_operator_apply(op.op.get(), a.data(), ra.data()));
  b200::check(rq_operator_apply(op.op.get(), b.data(), rb.data()));
  std::vector<cdouble> r(n2);
  for (long i = 0; i < n2; ++i) r[i] = {ra[i], rb[i]};
  if (ledger) ledger->add_fb(0);
  return r;
}

/// solve_quadratic: nev pairs nearest s.
inline std::vector<EigenPair> solve_quadratic(const QuadraticPencil& p, cdouble s, int nev, int m,
                                              double eps, CostLedger* ledger,
                                              std::uint64_t seed = 0, const Ordering* ord = nullptr) {
  Ordering local;
  if (!ord) fail(errc::config, "solve_quadratic needs the pencil's Ordering (nested_dissection_order)");
  const ShiftInvertOperator op = build_operator(p, s, *ord, ledger);
  rq_eigs_opts o{nev, m, eps, seed, 100, 1};
  std::vector<double> lr(nev), li(nev), res(nev), vr(op.n * nev), vi(op.n * nev);
  rq_eigs_info info{};
  const int rc = rq_eigs_run(op.op.get(), &o, lr.data(), li.data(), res.data(), vr.data(), vi.data(), &info);
  if (ledger) {
    for (std::int64_t k = 0; k < info.n_fb; ++k) ledger->add_fb(static_cast<std::uint64_t>(info.macs_fb / info.n_fb));
    for (std::int64_t k = 0; k < info.n_mv; ++k) ledger->add_mv(static_cast<std::uint64_t>(info.macs_mv / info.n_mv));
  }
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
