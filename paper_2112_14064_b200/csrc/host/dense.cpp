// SPDX-License-Identifier: Apache-2.0
#include "dense.hpp"

#include <algorithm>
#include <cmath>
#include <limits>

namespace rqb {

namespace {

// Givens pair (c real, s complex): c f + s g = r, -conj(s) f + c g = 0.
void givens(cplx f, cplx g, double& c, cplx& s) {
  const double af = std::abs(f), ag = std::abs(g);
  if (ag == 0.0) {
    c = 1.0;
    s = 0.0;
    return;
  }
  if (af == 0.0) {
    c = 0.0;
    s = std::conj(g) / ag;
    return;
  }
  const double r = std::hypot(af, ag);
  c = af / r;
  s = (f / af) * std::conj(g) / r;
}

// rows i, i+1 of T over columns [c0, c1): x' = c x + s y, y' = -conj(s) x + c y
void rot_rows(CMat& T, int i, int c0, int c1, double c, cplx s) {
  for (int j = c0; j < c1; ++j) {
    const cplx x = T(i, j), y = T(i + 1, j);
    T(i, j) = c * x + s * y;
    T(i + 1, j) = -std::conj(s) * x + c * y;
  }
}

// columns j, j+1 over rows [r0, r1): multiply on the right by G^H
void rot_cols(CMat& T, int j, int r0, int r1, double c, cplx s) {
  for (int i = r0; i < r1; ++i) {
    const cplx x = T(i, j), y = T(i, j + 1);
    T(i, j) = c * x + std::conj(s) * y;
    T(i, j + 1) = -s * x + c * y;
  }
}

}  // namespace

bool complex_schur(const std::vector<double>& A, int n, CMat& T, CMat& Z) {
  T = CMat(n);
  Z = CMat(n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) T(i, j) = A[i + static_cast<size_t>(j) * n];
  for (int i = 0; i < n; ++i) Z(i, i) = 1.0;
  // Householder reduction to upper Hessenberg form.
  std::vector<cplx> v(n);
  for (int k = 0; k + 2 < n; ++k) {
    double alpha2 = 0.0;
    for (int i = k + 1; i < n; ++i) alpha2 += std::norm(T(i, k));
    const double alpha = std::sqrt(alpha2);
    if (alpha == 0.0) continue;
    const cplx x0 = T(k + 1, k);
    const cplx ph = std::abs(x0) > 0 ? x0 / std::abs(x0) : cplx(1.0);
    for (int i = k + 1; i < n; ++i) v[i] = T(i, k);
    v[k + 1] += ph * alpha;
    double vn = 0.0;
    for (int i = k + 1; i < n; ++i) vn += std::norm(v[i]);
    if (vn == 0.0) continue;
    // T = (I - 2 v v^H / vn) T (I - 2 v v^H / vn)
    for (int j = 0; j < n; ++j) {
      cplx s = 0.0;
      for (int i = k + 1; i < n; ++i) s += std::conj(v[i]) * T(i, j);
      s *= 2.0 / vn;
      for (int i = k + 1; i < n; ++i) T(i, j) -= v[i] * s;
    }
    for (int i = 0; i < n; ++i) {
      cplx s = 0.0;
      for (int j = k + 1; j < n; ++j) s += T(i, j) * v[j];
      s *= 2.0 / vn;
      for (int j = k + 1; j < n; ++j) T(i, j) -= s * std::conj(v[j]);
    }
    for (int i = 0; i < n; ++i) {
      cplx s = 0.0;
      for (int j = k + 1; j < n; ++j) s += Z(i, j) * v[j];
      s *= 2.0 / vn;
      for (int j = k + 1; j < n; ++j) Z(i, j) -= s * std::conj(v[j]);
    }
    for (int i = k + 2; i < n; ++i) T(i, k) = 0.0;
  }
  // Single-shift complex QR.
  const double eps = std::numeric_limits<double>::epsilon();
  int ihi = n - 1, iter = 0, total = 0;
  while (ihi > 0) {
    int l = ihi;
    for (; l > 0; --l) {
      const double s = std::abs(T(l - 1, l - 1)) + std::abs(T(l, l));
      if (std::abs(T(l, l - 1)) <= eps * (s > 0 ? s : 1.0)) {
        T(l, l - 1) = 0.0;
        break;
      }
    }
    if (l == ihi) {
      --ihi;
      iter = 0;
      continue;
    }
    if (++total > 30 * n) return false;
    ++iter;
    cplx mu;
    if (iter % 11 == 10) {
      mu = T(ihi, ihi) + 0.75 * std::abs(T(ihi, ihi - 1));  // exceptional shift
    } else {
      const cplx a = T(ihi - 1, ihi - 1), b = T(ihi - 1, ihi), c = T(ihi, ihi - 1), d = T(ihi, ihi);
      const cplx half = 0.5 * (a - d);
      const cplx disc = std::sqrt(half * half + b * c);
      const cplx m1 = 0.5 * (a + d) + disc, m2 = 0.5 * (a + d) - disc;
      mu = std::abs(m1 - d) < std::abs(m2 - d) ? m1 : m2;
    }
    cplx x = T(l, l) - mu, y = T(l + 1, l);
    for (int k = l; k < ihi; ++k) {
      if (k > l) {
        x = T(k, k - 1);
        y = T(k + 1, k - 1);
      }
      double c;
      cplx s;
      givens(x, y, c, s);
      rot_rows(T, k, k > l ? k - 1 : k, n, c, s);
      if (k > l) T(k + 1, k - 1) = 0.0;
      rot_cols(T, k, 0, std::min(k + 3, ihi + 1), c, s);
      rot_cols(Z, k, 0, n, c, s);
    }
  }
  for (int j = 0; j < n; ++j)
    for (int i = j + 1; i < n; ++i) T(i, j) = 0.0;
  return true;
}

void schur_reorder(CMat& T, CMat& Z, std::vector<int>& sel) {
  const int n = T.n;
  int ks = 0;
  for (int k = 0; k < n; ++k) {
    if (!sel[k]) continue;
    for (int j = k - 1; j >= ks; --j) {
      // swap diagonal entries j, j+1
      const cplx t11 = T(j, j), t22 = T(j + 1, j + 1);
      double c;
      cplx s;
      givens(T(j, j + 1), t22 - t11, c, s);
      rot_rows(T, j, j + 2, n, c, s);
      rot_cols(T, j, 0, j, c, s);
      // columns: x' = c x + conj(s) y, y' = -s x + c y  (zrot with conj(sn))
      T(j, j) = t22;
      T(j + 1, j + 1) = t11;
      rot_cols(Z, j, 0, n, c, s);
      std::swap(sel[j], sel[j + 1]);
    }
    ++ks;
  }
}

CMat triangular_eigvecs(const CMat& T) {
  const int n = T.n;
  CMat Y(n);
  double tnorm = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i <= j; ++i) tnorm = std::max(tnorm, std::abs(T(i, j)));
  const double smin = std::max(tnorm * std::numeric_limits<double>::epsilon(), 1e-300);
  for (int j = 0; j < n; ++j) {
    Y(j, j) = 1.0;
    const cplx lam = T(j, j);
    for (int i = j - 1; i >= 0; --i) {
      cplx s = 0.0;
      for (int t = i + 1; t <= j; ++t) s += T(i, t) * Y(t, j);
      cplx den = T(i, i) - lam;
      if (std::abs(den) < smin) den = smin;
      Y(i, j) = -s / den;
    }
    double nrm = 0.0;
    for (int i = 0; i <= j; ++i) nrm += std::norm(Y(i, j));
    nrm = std::sqrt(nrm);
    for (int i = 0; i <= j; ++i) Y(i, j) /= nrm;
  }
  return Y;
}

int real_basis(const CMat& Z, int p, std::vector<double>& Q) {
  const int n = Z.n;
  std::vector<std::vector<double>> cols;
  cols.reserve(2 * p);
  for (int j = 0; j < p; ++j) {
    std::vector<double> re(n), im(n);
    for (int i = 0; i < n; ++i) re[i] = Z(i, j).real(), im[i] = Z(i, j).imag();
    cols.push_back(std::move(re));
    cols.push_back(std::move(im));
  }
  Q.assign(static_cast<size_t>(n) * p, 0.0);
  std::vector<char> used(cols.size(), 0);
  int rank = 0;
  double maxn0 = 0.0;
  for (auto& c : cols) {
    double s = 0;
    for (double x : c) s += x * x;
    maxn0 = std::max(maxn0, std::sqrt(s));
  }
  while (rank < p) {
    int best = -1;
    double bn = 0.0;
    for (size_t j = 0; j < cols.size(); ++j) {
      if (used[j]) continue;
      double s = 0;
      for (double x : cols[j]) s += x * x;
      if (s > bn) bn = s, best = static_cast<int>(j);
    }
    if (best < 0 || std::sqrt(bn) <= 1e-10 * maxn0) break;
    used[best] = 1;
    std::vector<double> q = cols[best];
    for (int pass = 0; pass < 2; ++pass)
      for (int r = 0; r < rank; ++r) {
        double d = 0;
        for (int i = 0; i < n; ++i) d += Q[i + static_cast<size_t>(r) * n] * q[i];
        for (int i = 0; i < n; ++i) q[i] -= d * Q[i + static_cast<size_t>(r) * n];
      }
    double s = 0;
    for (double x : q) s += x * x;
    s = std::sqrt(s);
    if (s <= 1e-12 * maxn0) continue;
    for (int i = 0; i < n; ++i) Q[i + static_cast<size_t>(rank) * n] = q[i] / s;
    ++rank;
    // deflate remaining candidates
    for (size_t j = 0; j < cols.size(); ++j) {
      if (used[j]) continue;
      double d = 0;
      for (int i = 0; i < n; ++i) d += Q[i + static_cast<size_t>(rank - 1) * n] * cols[j][i];
      for (int i = 0; i < n; ++i) cols[j][i] -= d * Q[i + static_cast<size_t>(rank - 1) * n];
    }
  }
  return rank;
}

}  // namespace rqb
