// CPU unit test of the host dense kernels used by the Krylov-Schur driver
// (paper_2112_14064_b200/csrc/host/dense.cpp): Schur form, reordering, real
// basis of a conjugation-closed invariant subspace.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>

#include "../../paper_2112_14064_b200/csrc/host/dense.hpp"

using namespace rqb;

int main() {
  std::mt19937_64 g(1);
  std::normal_distribution<double> N;
  int fails = 0;
  const std::pair<int, bool> cases[] = {{2, false}, {5, false}, {21, false}, {41, false}, {80, false},
                                         {40, true}, {41, true}};
  for (const auto& cs : cases) {
    const int n = cs.first;
    std::vector<double> A(n * n);
    for (auto& x : A) x = N(g);
    if (cs.second) {
      // degenerate cluster: Q blockdiag([a b; -b a] x k (+ one real)) Q^T
      // with a random orthogonal Q (repeated complex pair, as in the QEP)
      std::vector<double> D(n * n, 0.0), Q(n * n);
      for (int i = 0; i + 1 < n; i += 2) {
        D[i + i * n] = D[(i + 1) + (i + 1) * n] = -0.03;
        D[i + (i + 1) * n] = 0.9995;
        D[(i + 1) + i * n] = -0.9995;
      }
      if (n % 2) D[(n - 1) * (n + 1)] = 0.5;
      for (auto& x : Q) x = N(g);
      for (int j = 0; j < n; ++j) {  // MGS -> orthogonal
        for (int t = 0; t < j; ++t) {
          double d = 0;
          for (int i = 0; i < n; ++i) d += Q[i + t * n] * Q[i + j * n];
          for (int i = 0; i < n; ++i) Q[i + j * n] -= d * Q[i + t * n];
        }
        double nr = 0;
        for (int i = 0; i < n; ++i) nr += Q[i + j * n] * Q[i + j * n];
        for (int i = 0; i < n; ++i) Q[i + j * n] /= std::sqrt(nr);
      }
      std::vector<double> QD(n * n, 0.0);
      for (int j = 0; j < n; ++j) for (int t = 0; t < n; ++t) for (int i = 0; i < n; ++i)
        QD[i + j * n] += Q[i + t * n] * D[t + j * n];
      std::fill(A.begin(), A.end(), 0.0);
      for (int j = 0; j < n; ++j) for (int t = 0; t < n; ++t) for (int i = 0; i < n; ++i)
        A[i + j * n] += QD[i + t * n] * Q[j + t * n];
    }
    CMat T, Z;
    if (!complex_schur(A, n, T, Z)) { std::printf("qr fail n=%d\n", n); return 1; }
    auto defect = [&](const CMat& T, const CMat& Z) {
      double d = 0;
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          cplx s = 0;  // (Z T Z^H)(i,j)
          for (int a = 0; a < n; ++a)
            for (int b = a; b < n; ++b) s += Z(i, a) * T(a, b) * std::conj(Z(j, b));
          d = std::max(d, std::abs(s - A[i + j * n]));
        }
      return d;
    };
    const double d0 = defect(T, Z);
    // select eigenvalues with the largest modulus, closed under conjugation
    std::vector<int> sel(n, 0);
    std::vector<std::pair<double, int>> ord;
    for (int i = 0; i < n; ++i) ord.push_back({-std::abs(T(i, i)), i});
    std::sort(ord.begin(), ord.end());
    int want = n / 2, p = 0;
    for (auto& o : ord) {
      if (p >= want) break;
      const int i = o.second;
      if (sel[i]) continue;
      sel[i] = 1; ++p;
      if (std::abs(T(i, i).imag()) > 1e-12) {
        int best = -1; double bd = 1e300;
        for (int q = 0; q < n; ++q) if (!sel[q]) {
          double d = std::abs(T(q, q) - std::conj(T(i, i)));
          if (d < bd) bd = d, best = q;
        }
        sel[best] = 1; ++p;
      }
    }
    std::vector<int> s2 = sel;
    schur_reorder(T, Z, s2);
    const double d1 = defect(T, Z);
    bool lead = true;
    for (int i = 0; i < n; ++i) if (s2[i] != (i < p)) lead = false;
    std::vector<double> Q;
    const int rank = real_basis(Z, p, Q);
    // invariance of span(Q): A Q = Q (Q^T A Q)
    double inv = 0;
    std::vector<double> AQ(n * p, 0.0), Tq(p * p, 0.0);
    for (int c = 0; c < p; ++c) for (int t = 0; t < n; ++t) for (int i = 0; i < n; ++i)
      AQ[i + c * n] += A[i + t * n] * Q[t + c * n];
    for (int c = 0; c < p; ++c) for (int i = 0; i < p; ++i) for (int t = 0; t < n; ++t)
      Tq[i + c * p] += Q[t + i * n] * AQ[t + c * n];
    for (int c = 0; c < p; ++c) for (int i = 0; i < n; ++i) {
      double s = AQ[i + c * n];
      for (int t = 0; t < p; ++t) s -= Q[i + t * n] * Tq[t + c * p];
      inv = std::max(inv, std::fabs(s));
    }
    const bool ok = d0 < 1e-12 * n && d1 < 1e-12 * n && lead && rank == p && inv < 1e-11 * n;
    std::printf("n=%d%s p=%d schur=%.2e reorder=%.2e rank=%d invariance=%.2e %s\n", n, cs.second ? " (degenerate)" : "", p, d0, d1, rank,
                inv, ok ? "ok" : "FAIL");
    fails += !ok;
    // the same selection on the real Schur form (real_schur_reorder): A Zr =
    // Zr Tr, Zr orthogonal, Tr block upper triangular with the selected part
    // leading (T[p.., :p] = 0) and its eigenvalues the selected ones
    std::vector<double> Tr, Zr;
    if (!real_schur(A, n, Tr, Zr)) { std::printf("real qr fail n=%d\n", n); return 1; }
    CMat Tc, Zc;
    complexify_schur(Tr, Zr, n, Tc, Zc);
    std::vector<cplx> want_ev;
    for (int i = 0; i < n; ++i) if (sel[i]) want_ev.push_back(Tc(i, i));
    std::vector<int> s3 = sel;
    const int pr = real_schur_reorder(Tr, Zr, n, s3);
    double rd = 0, ro = 0, an = 0, low = 0;
    for (double x : A) an = std::max(an, std::fabs(x));
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double s = 0, o = 0;
        for (int t = 0; t < n; ++t) {
          s += A[i + t * n] * Zr[t + j * n] - Zr[i + t * n] * Tr[t + j * n];
          o += Zr[t + i * n] * Zr[t + j * n];
        }
        rd = std::max(rd, std::fabs(s));
        ro = std::max(ro, std::fabs(o - (i == j ? 1.0 : 0.0)));
        if (i > j + 1 || (j < pr && i >= pr)) low = std::max(low, std::fabs(Tr[i + j * n]));
      }
    std::vector<cplx> got_ev;  // eigenvalues of the leading pr x pr blocks
    for (int k = 0; k < pr; ++k) {
      if (k + 1 < pr && Tr[(k + 1) + k * n] != 0.0) {
        const double a = Tr[k + k * n], b = Tr[k + (k + 1) * n], c = Tr[(k + 1) + k * n], d = Tr[(k + 1) + (k + 1) * n];
        const cplx h = 0.5 * (a + d), q = std::sqrt(cplx(0.25 * (a - d) * (a - d) + b * c));
        got_ev.push_back(h + q);
        got_ev.push_back(h - q);
        ++k;
      } else {
        got_ev.push_back(Tr[k + k * n]);
      }
    }
    // every selected eigenvalue is among the leading ones (the leading part
    // may hold more: a selected pair member closes its 2 x 2 block)
    double evd = 0;
    std::vector<int> used(got_ev.size(), 0);
    for (const cplx& w : want_ev) {
      double bd = 1e300;
      int bi = -1;
      for (size_t q = 0; q < got_ev.size(); ++q)
        if (!used[q] && std::abs(got_ev[q] - w) < bd) bd = std::abs(got_ev[q] - w), bi = static_cast<int>(q);
      if (bi >= 0) used[bi] = 1;
      evd = std::max(evd, bd / std::max(1.0, std::abs(w)));
    }
    const bool rok = pr >= p && (cs.second || pr == p) && rd < 1e-12 * n * std::max(1.0, an) && ro < 1e-12 * n &&
                     low == 0.0 && evd < 1e-8;
    std::printf("real reorder n=%d p=%d: defect %.2e orth %.2e below %.1e ev %.1e %s\n", n, pr, rd, ro, low, evd,
                rok ? "rok" : "rFAIL");
    fails += !rok;
  }
    // complex input (complex_schur_c): random complex matrices
  for (int n : {1, 2, 7, 40, 121}) {
    CMat A(n);
    for (auto& z : A.a) z = cplx(N(g), N(g));
    CMat T, Z;
    if (!complex_schur_c(A, T, Z)) { std::printf("zqr fail n=%d\n", n); return 1; }
    double d = 0, u = 0, l = 0, an = 0;
    for (const auto& z : A.a) an = std::max(an, std::abs(z));
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        cplx sacc = 0, zz = 0;
        for (int a = 0; a < n; ++a) {
          zz += std::conj(Z(a, i)) * Z(a, j);
          for (int b2 = a; b2 < n; ++b2) sacc += Z(i, a) * T(a, b2) * std::conj(Z(j, b2));
        }
        d = std::max(d, std::abs(sacc - A(i, j)));
        u = std::max(u, std::abs(zz - (i == j ? 1.0 : 0.0)));
        if (i > j) l = std::max(l, std::abs(T(i, j)));
      }
    const bool ok = d <= 1e-12 * std::max(1.0, an) * n && u <= 1e-12 * n && l == 0.0;
    std::printf("complex n=%d defect %.2e unitarity %.2e %s\n", n, d, u, ok ? "zok" : "zFAIL");
    if (!ok) ++fails;
  }
  return fails;
}
