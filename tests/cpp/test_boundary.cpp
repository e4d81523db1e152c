// SPDX-License-Identifier: Apache-2.0
// The C++ drop-in surface (include/rigaqep/{sparsela,eig}.hpp) linked the way
// a reference build would link it: the reference's own types and sources
// (proj/include, splines.cpp / spaces.cpp / sparse.cpp / kernels*.cpp,
// compiled from /root/reference by oracle/Makefile) plus librq_b200.so.
// Built by __graft_entry__.build() (tests/cpp/Makefile); run by
// tests/test_boundary_cpp.py on a GPU. Prints one JSON line of results and
// exits non-zero on the first failed check.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "rigaqep/eig.hpp"
#include "rigaqep/sparsela.hpp"
#include "rigaqep/spaces.hpp"

namespace {

int g_checks = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(cond)) {                                                               \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
      std::exit(1);                                                              \
    }                                                                            \
  } while (0)

rq::SparseMatrix csr(long n, const std::vector<std::int64_t>& rp, const std::vector<std::int32_t>& col,
                     const std::vector<double>& v) {
  rq::SparseMatrix a;
  a.n = n;
  a.rowptr = rp;
  a.col = col;
  a.val.resize(v.size());
  for (std::size_t k = 0; k < v.size(); ++k) a.val[k] = v[k];
  return a;
}

rq::SparseMatrix diag(const std::vector<double>& d) {
  std::vector<std::int64_t> rp(d.size() + 1);
  std::vector<std::int32_t> col(d.size());
  for (std::size_t i = 0; i < d.size(); ++i) rp[i + 1] = static_cast<std::int64_t>(i + 1), col[i] = static_cast<std::int32_t>(i);
  return csr(static_cast<long>(d.size()), rp, col, d);
}

double splitmix_uniform(std::uint64_t& s) {
  std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (static_cast<double>(z >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
}

}  // namespace

int main() {
  // ---- cfg1 (BASELINE configs[0]): H(div) p=2 32^2 IGA on the reference's space
  const rq::VectorSpace vs = rq::build_iga_space(rq::SpaceKind::divergence, 2, 32, rq::BoxGeometry{});
  const std::vector<long> cons = rq::boundary_mask(vs, rq::ModelProblem::acoustic);
  rq_space_desc d{RQ_SPACE_DIV, 2, 32, 0, 0.05, 0.01};
  rq_pencil_t* ph = nullptr;
  rq::b200::check(rq_pencil_assemble(&d, &ph));
  std::int64_t nfull, n, nnz;
  rq::b200::check(rq_pencil_dims(ph, &nfull, &n, &nnz));
  CHECK(nfull == vs.N() && n == vs.N() - static_cast<long>(cons.size()));
  std::vector<std::int64_t> rp(n + 1);
  std::vector<std::int32_t> col(nnz);
  std::vector<double> K(nnz), C(nnz), M(nnz);
  rq::b200::check(rq_pencil_csr(ph, rp.data(), col.data(), K.data(), C.data(), M.data()));
  rq_pencil_destroy(ph);
  rq::QuadraticPencil P = rq::make_pencil(vs, cons, csr(n, rp, col, K), csr(n, rp, col, C), csr(n, rp, col, M));
  CHECK(P.ordering->method == "geometric-nested-dissection" && P.ordering->n() == n);

  // ---- build_operator / apply_operator / b_inner / arnoldi_run / ritz_extract / restart
  rq::CostLedger L;
  L.flops_per_mac = 2.0;  // real arithmetic on the GPU path
  const rq::ShiftInvertOperator op = rq::build_operator(P, {-0.5, 0.0}, *P.ordering, &L);
  CHECK(L.fa_ops() == 1 && L.fa_macs() > 0);
  std::vector<rq::cdouble> v(2 * n);
  std::uint64_t seed = 0;
  for (auto& z : v) z = splitmix_uniform(seed);
  const std::vector<rq::cdouble> r = rq::apply_operator(op, v, &L);
  CHECK(L.fb_ops() == 1 && L.mv_ops() == 3 && L.vv_ops() == 3);
  // r_l = s r_u + v_u
  double dl = 0;
  for (long i = 0; i < n; ++i) dl = std::max(dl, std::abs(r[n + i] - (-0.5 * r[i] + v[i])));
  CHECK(dl <= 1e-12 * (1.0 + std::abs(r[0])));
  // complex input: two real applications, charged as one operation
  std::vector<rq::cdouble> vc(v);
  for (auto& z : vc) z *= rq::cdouble(0.6, 0.8);
  const std::vector<rq::cdouble> rc = rq::apply_operator(op, vc, &L);
  double dc = 0, sc = 0;
  for (long i = 0; i < 2 * n; ++i) dc = std::max(dc, std::abs(rc[i] - rq::cdouble(0.6, 0.8) * r[i])), sc = std::max(sc, std::abs(r[i]));
  CHECK(dc <= 1e-12 * sc && L.fb_ops() == 2);
  const rq::cdouble bi = rq::b_inner(op, v, v, &L);
  CHECK(bi.real() > 0 && bi.imag() == 0.0 && L.mv_ops() == 7);

  const int m = 21;
  rq::KrylovState S = rq::arnoldi_run(op, P.M, m, v, &L);
  CHECK(S.m == m && static_cast<int>(S.V.size()) == m + 1 && S.beta > 0);
  // B-orthonormality of the basis, B = diag(I, M)
  double orth = 0;
  for (int i = 0; i <= m; i += 5)
    for (int j = 0; j <= m; j += 4) {
      std::vector<rq::cdouble> ml(n), mv(n);
      rq::spmv(P.M, std::vector<rq::cdouble>(S.V[j].begin() + n, S.V[j].end()), ml, nullptr);
      rq::cdouble g = 0;
      for (long k = 0; k < n; ++k) g += std::conj(S.V[i][k]) * S.V[j][k] + std::conj(S.V[i][n + k]) * ml[k];
      orth = std::max(orth, std::abs(g - (i == j ? 1.0 : 0.0)));
    }
  CHECK(orth <= 1e-8);
  const std::vector<rq::RitzValue> rz = rq::ritz_extract(S, op);
  CHECK(static_cast<int>(rz.size()) == m);
  for (int a = 1; a < m; ++a) CHECK(std::abs(rz[a].lambda + 0.5) >= std::abs(rz[a - 1].lambda + 0.5) * (1 - 1e-12));
  const rq::KrylovState R = rq::krylov_schur_restart(op, S, 10, 11, &L);
  CHECK((R.m == 11 || R.m == 12) && L.restart_ops() == 1);

  // ---- solve_quadratic (SPEC.md:462 signature; the pencil's ordering)
  rq::CostLedger L2;
  L2.flops_per_mac = 2.0;
  const std::vector<rq::EigenPair> pairs = rq::solve_quadratic(P, {-0.5, 0.0}, 10, 21, 1e-10, &L2);
  const rq::cdouble cl(-0.03, std::sqrt(0.9991));
  double worst = 0, dist = 0;
  for (const auto& e : pairs) {
    worst = std::max(worst, e.residual);
    dist = std::max(dist, std::min(std::abs(e.lambda - cl), std::abs(e.lambda - std::conj(cl))));
  }
  CHECK(worst <= 1e-10 && dist <= 1e-8);
  CHECK(L2.fa_ops() == 1 && L2.fb_ops() > 0 && L2.restart_ops() > 0 && L2.check_ops() >= 10);
  CHECK(L2.mv_ops() >= 6 * L2.fb_ops() && L2.mv_ops() <= 6 * L2.fb_ops() + 2 * L2.fb_ops() / 10 + 8);

  // ---- SPEC's hand examples on the natural ordering (no space attached)
  {  // K = diag(1, 4, 9), C = 0, M = I, s = 0.1: the two nearest are +-i
    rq::QuadraticPencil Q{diag({1, 4, 9}), diag({0, 0, 0}), diag({1, 1, 1}), nullptr};
    const auto e = rq::solve_quadratic(Q, {0.1, 0.0}, 2, 4, 1e-10, nullptr);
    double err = 0;
    for (const auto& x : e) err = std::max(err, std::min(std::abs(x.lambda - rq::cdouble(0, 1)), std::abs(x.lambda - rq::cdouble(0, -1))));
    CHECK(err <= 1e-10 && std::abs(e[0].lambda.imag() + e[1].lambda.imag()) <= 1e-10);
  }
  {  // scale_pencil known answer: K = 4I, C = M = I -> varsigma = 2
    rq::QuadraticPencil Q{diag({4, 4, 4}), diag({1, 1, 1}), diag({1, 1, 1}), nullptr};
    const auto sp = rq::scale_pencil(Q);
    CHECK(sp.second == 2.0 && sp.first.C.val[0] == 2.0 && sp.first.M.val[1] == 4.0 && sp.first.varsigma == 2.0);
  }
  {  // dense 3x3 LU known answer: [[4,3,0],[6,3,1],[0,1,2]]
    const rq::SparseMatrix A = csr(3, {0, 3, 6, 9}, {0, 1, 2, 0, 1, 2, 0, 1, 2}, {4, 3, 0, 6, 3, 1, 0, 1, 2});
    rq::CostLedger L3;
    const rq::Factorization F = rq::lu_factorize(A, rq::natural_order(3), &L3);
    const auto x = rq::solve_factored(F, {1.0, 2.0, 3.0}, &L3);
    std::vector<rq::cdouble> Ax(3);
    rq::spmv(A, x, Ax, nullptr);
    CHECK(std::abs(Ax[0] - 1.0) <= 1e-14 && std::abs(Ax[1] - 2.0) <= 1e-14 && std::abs(Ax[2] - 3.0) <= 1e-14);
    CHECK(L3.fa_ops() == 1 && L3.fa_macs() == 4 + 1 && L3.fb_ops() == 1);  // (3-1)^2 + (3-2)^2 MACs
  }
  {  // complex A (complex shift): Q(-0.5 + 0.3i) of the cfg1 pencil, real-equivalent GPU LU
    const rq::cdouble sc(-0.5, 0.3);
    rq::SparseMatrix Q = P.K;
    for (std::size_t k = 0; k < Q.val.size(); ++k) Q.val[k] = P.K.val[k] + sc * P.C.val[k] + sc * sc * P.M.val[k];
    const rq::Factorization Fc = rq::lu_factorize(Q, *P.ordering, nullptr);
    std::vector<rq::cdouble> bc(n), Qx(n);
    for (long i = 0; i < n; ++i) bc[i] = rq::cdouble(std::sin(0.3 * i), std::cos(0.7 * i));
    const auto xc = rq::solve_factored(Fc, bc, nullptr);
    rq::spmv(Q, xc, Qx, nullptr);
    double rmax = 0, xmax = 0;
    for (long i = 0; i < n; ++i) rmax = std::max(rmax, std::abs(Qx[i] - bc[i])), xmax = std::max(xmax, std::abs(xc[i]));
    CHECK(Fc.complex_values && rmax <= 1e-10 * std::max(1.0, xmax));
  }
  // ---- error behaviour: reference error categories through the boundary
  bool threw = false;
  try {
    rq::build_operator(P, {-0.5, 0.1}, *P.ordering, nullptr);
  } catch (const rq::Error& e) {
    threw = e.code() == rq::errc::config;
  }
  CHECK(threw);
  threw = false;
  try {
    rq::apply_operator(op, std::vector<rq::cdouble>(3), nullptr);
  } catch (const rq::Error& e) {
    threw = e.code() == rq::errc::dimension;
  }
  CHECK(threw);

  std::printf("{\"checks\": %d, \"ledger_json\": %s, \"solve_ledger_json\": %s}\n", g_checks,
              [&] { std::string s = L.to_json(); for (char& c : s) if (c == '\n') c = ' '; return s; }().c_str(),
              [&] { std::string s = L2.to_json(); for (char& c : s) if (c == '\n') c = ' '; return s; }().c_str());
  return 0;
}
