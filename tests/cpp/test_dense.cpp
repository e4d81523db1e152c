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
  for (int n : {2, 5, 21, 41, 80}) {
    std::vector<double> A(n * n);
    for (auto& x : A) x = N(g);
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
    std::printf("n=%d p=%d schur=%.2e reorder=%.2e rank=%d invariance=%.2e %s\n", n, p, d0, d1, rank,
                inv, ok ? "ok" : "FAIL");
    fails += !ok;
  }
  return fails;
}
