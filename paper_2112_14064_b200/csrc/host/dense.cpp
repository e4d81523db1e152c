// SPDX-License-Identifier: Apache-2.0
#include "dense.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <thread>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "common.hpp"

namespace rqb {

int host_threads() {
#ifdef _OPENMP
  static const int t = std::max(1, std::min(8, omp_get_num_procs() / 2));
#else
  static const int t = 1;
#endif
  return t;
}

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

namespace {

// Householder reduction of the real n x n matrix H (column-major) to upper
// Hessenberg form, H <- Q^T H Q, Zr <- Zr Q. Columns whose entries below the
// subdiagonal are already zero (the Arnoldi part of a Krylov-Schur matrix)
// are skipped; reflectors stop at the column's last nonzero row.
void hessenberg_real(std::vector<double>& Hv, std::vector<double>& Zv, int n) {
  auto H = [&](int i, int j) -> double& { return Hv[i + static_cast<size_t>(j) * n]; };
  std::vector<double> v(n), w(n);
  for (int k = 0; k + 2 < n; ++k) {
    int e = n - 1;
    while (e > k + 1 && H(e, k) == 0.0) --e;
    if (e == k + 1) continue;
    double alpha2 = 0.0;
    for (int i = k + 1; i <= e; ++i) alpha2 += H(i, k) * H(i, k);
    const double x0 = H(k + 1, k);
    const double beta = -std::copysign(std::sqrt(alpha2), x0);
    v[k + 1] = x0 - beta;
    double vtv = v[k + 1] * v[k + 1];
    for (int i = k + 2; i <= e; ++i) v[i] = H(i, k), vtv += v[i] * v[i];
    const double tau = 2.0 / vtv;
    // left: rows k+1..e of columns k+1..n-1; column k becomes beta e_1
    H(k + 1, k) = beta;
    for (int i = k + 2; i <= e; ++i) H(i, k) = 0.0;
    for (int j = k + 1; j < n; ++j) {
      double* col = &H(0, j);
      double sdot = 0.0;
      for (int i = k + 1; i <= e; ++i) sdot += v[i] * col[i];
      sdot *= tau;
      for (int i = k + 1; i <= e; ++i) col[i] -= sdot * v[i];
    }
    // right: columns k+1..e of H (all rows) and of Zr
    for (double* M : {Hv.data(), Zv.data()}) {
      std::fill(w.begin(), w.end(), 0.0);
      for (int j = k + 1; j <= e; ++j) {
        const double* col = M + static_cast<size_t>(j) * n;
        const double vj = v[j];
        for (int i = 0; i < n; ++i) w[i] += col[i] * vj;
      }
      for (int j = k + 1; j <= e; ++j) {
        double* col = M + static_cast<size_t>(j) * n;
        const double f = tau * v[j];
        for (int i = 0; i < n; ++i) col[i] -= f * w[i];
      }
    }
  }
}

// Francis double-shift QR of the real upper Hessenberg H to quasi-triangular
// (real Schur) form, accumulating Zr; real eigenvalue pairs are split by a
// rotation, complex pairs stay 2 x 2 blocks. Returns false if more than 30 n
// iterations were needed.
bool francis_real(std::vector<double>& Hv, std::vector<double>& Zv, int n) {
  auto H = [&](int i, int j) -> double& { return Hv[i + static_cast<size_t>(j) * n]; };
  const double eps = std::numeric_limits<double>::epsilon();
  double anorm = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i <= std::min(j + 1, n - 1); ++i) anorm += std::fabs(H(i, j));
  if (anorm == 0.0) anorm = 1.0;
  // rotation [c -s; s c] on rows/columns (k, k+1) that zeroes H(k+1, k) of a
  // 2 x 2 block with real eigenvalues
  auto split_real_pair = [&](int k) {
    const double p = 0.5 * (H(k, k) - H(k + 1, k + 1));
    const double q = p * p + H(k + 1, k) * H(k, k + 1);
    if (q < 0.0) return;  // complex pair: stays a 2 x 2 block
    const double zz = p + std::copysign(std::sqrt(q), p);
    const double x = H(k + 1, k);
    const double sc = std::fabs(x) + std::fabs(zz);
    if (sc == 0.0) return;
    double pp = x / sc, qq = zz / sc;
    const double r = std::sqrt(pp * pp + qq * qq);
    pp /= r;
    qq /= r;
    for (int j = k; j < n; ++j) {
      const double t = H(k, j);
      H(k, j) = qq * t + pp * H(k + 1, j);
      H(k + 1, j) = qq * H(k + 1, j) - pp * t;
    }
    for (double* M : {Hv.data(), Zv.data()}) {
      const int rows = M == Hv.data() ? k + 2 : n;
      double* c0 = M + static_cast<size_t>(k) * n;
      double* c1 = c0 + n;
      for (int i = 0; i < rows; ++i) {
        const double t = c0[i];
        c0[i] = qq * t + pp * c1[i];
        c1[i] = qq * c1[i] - pp * t;
      }
    }
    H(k + 1, k) = 0.0;
  };
  int nn = n - 1, its = 0, total = 0;
  while (nn >= 0) {
    int l = nn;
    for (; l > 0; --l) {
      double s = std::fabs(H(l - 1, l - 1)) + std::fabs(H(l, l));
      if (s == 0.0) s = anorm;
      if (std::fabs(H(l, l - 1)) <= eps * s) {
        H(l, l - 1) = 0.0;
        break;
      }
    }
    if (l == nn) {  // one eigenvalue
      --nn;
      its = 0;
      continue;
    }
    if (l == nn - 1) {  // a 2 x 2 block
      split_real_pair(nn - 1);
      nn -= 2;
      its = 0;
      continue;
    }
    if (++total > 30 * n) return false;
    ++its;
    // shifts: eigenvalues of the trailing 2 x 2 (trace x + y, x y - w); an
    // exceptional shift every 10 iterations without deflation
    double x = H(nn, nn), y = H(nn - 1, nn - 1), w = H(nn, nn - 1) * H(nn - 1, nn);
    if (its % 10 == 0) {
      const double s = std::fabs(H(nn, nn - 1)) + std::fabs(H(nn - 1, nn - 2));
      x = y = H(nn, nn) + 0.75 * s;
      w = -0.4375 * s * s;
    }
    // first column of (H - s1)(H - s2), started at the lowest row m where two
    // consecutive small subdiagonals allow it
    int m = nn - 2;
    double p = 0, q = 0, r = 0;
    for (; m >= l; --m) {
      const double z = H(m, m);
      const double rr = x - z, ss = y - z;
      p = (rr * ss - w) / H(m + 1, m) + H(m, m + 1);
      q = H(m + 1, m + 1) - z - rr - ss;
      r = H(m + 2, m + 1);
      const double sc = std::fabs(p) + std::fabs(q) + std::fabs(r);
      p /= sc;
      q /= sc;
      r /= sc;
      if (m == l) break;
      const double u = std::fabs(H(m, m - 1)) * (std::fabs(q) + std::fabs(r));
      const double v = std::fabs(p) * (std::fabs(H(m - 1, m - 1)) + std::fabs(z) + std::fabs(H(m + 1, m + 1)));
      if (u <= eps * v) break;
    }
    for (int i = m + 2; i <= nn; ++i) {
      H(i, i - 2) = 0.0;
      if (i != m + 2) H(i, i - 3) = 0.0;
    }
    // bulge chase with 3-element reflectors (2-element at the bottom)
    for (int k = m; k <= nn - 1; ++k) {
      const bool three = k != nn - 1;
      double sc = 1.0;
      if (k != m) {
        p = H(k, k - 1);
        q = H(k + 1, k - 1);
        r = three ? H(k + 2, k - 1) : 0.0;
        sc = std::fabs(p) + std::fabs(q) + std::fabs(r);
        if (sc == 0.0) continue;
        p /= sc;
        q /= sc;
        r /= sc;
      }
      const double s = std::copysign(std::sqrt(p * p + q * q + r * r), p);
      if (s == 0.0) continue;
      if (k == m) {
        if (l != m) H(k, k - 1) = -H(k, k - 1);
      } else {
        H(k, k - 1) = -s * sc;
        H(k + 1, k - 1) = 0.0;
        if (three) H(k + 2, k - 1) = 0.0;
      }
      p += s;
      const double vx = p / s, vy = q / s, vz = r / s;
      q /= p;
      r /= p;
      for (int j = k; j < n; ++j) {
        double* col = &H(0, j);
        double t = col[k] + q * col[k + 1];
        if (three) {
          t += r * col[k + 2];
          col[k + 2] -= t * vz;
        }
        col[k + 1] -= t * vy;
        col[k] -= t * vx;
      }
      for (double* M : {Hv.data(), Zv.data()}) {
        const int rows = M == Hv.data() ? std::min(nn, k + 3) + 1 : n;
        double* c0 = M + static_cast<size_t>(k) * n;
        double* c1 = c0 + n;
        double* c2 = c1 + n;
        if (three) {
          for (int i = 0; i < rows; ++i) {
            const double t = vx * c0[i] + vy * c1[i] + vz * c2[i];
            c2[i] -= t * r;
            c1[i] -= t * q;
            c0[i] -= t;
          }
        } else {
          for (int i = 0; i < rows; ++i) {
            const double t = vx * c0[i] + vy * c1[i];
            c1[i] -= t * q;
            c0[i] -= t;
          }
        }
      }
    }
  }
  for (int j = 0; j < n; ++j)
    for (int i = j + 2; i < n; ++i) H(i, j) = 0.0;
  return true;
}

}  // namespace

bool real_schur(const std::vector<double>& A, int n, std::vector<double>& T, std::vector<double>& Z) {
  T.assign(A.begin(), A.begin() + static_cast<size_t>(n) * n);
  Z.assign(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i) Z[i + static_cast<size_t>(i) * n] = 1.0;
  hessenberg_real(T, Z, n);
  return francis_real(T, Z, n);
}

// Each 2 x 2 block (a complex-conjugate pair) of the real Schur form is
// triangularised by one complex rotation: A = Z T Z^H with T upper triangular.
void complexify_schur(const std::vector<double>& H, const std::vector<double>& Zr, int n, CMat& T, CMat& Z) {
  T = CMat(n);
  Z = CMat(n);
  for (size_t i = 0; i < H.size(); ++i) {
    T.a[i] = H[i];
    Z.a[i] = Zr[i];
  }
  for (int k = 0; k + 1 < n; ++k) {
    if (T(k + 1, k) == 0.0) continue;
    const cplx a = T(k, k), b = T(k, k + 1), c = T(k + 1, k), d = T(k + 1, k + 1);
    const cplx p = 0.5 * (a - d);
    const cplx mu_d = p + std::sqrt(p * p + b * c);  // mu - d for one eigenvalue mu of the block
    const double r = std::hypot(std::abs(mu_d), std::abs(c));
    const cplx cs = mu_d / r, sn = c / r;  // G = [conj(cs) sn; -sn cs] (sn real)
    for (int j = k; j < n; ++j) {
      const cplx x = T(k, j), y = T(k + 1, j);
      T(k, j) = std::conj(cs) * x + sn * y;
      T(k + 1, j) = -sn * x + cs * y;
    }
    auto right = [&](CMat& M, int rows) {  // M[:, k:k+2] *= G^H
      for (int i = 0; i < rows; ++i) {
        const cplx x = M(i, k), y = M(i, k + 1);
        M(i, k) = cs * x + std::conj(sn) * y;
        M(i, k + 1) = -sn * x + std::conj(cs) * y;
      }
    };
    right(T, k + 2);
    right(Z, n);
    T(k + 1, k) = 0.0;
    ++k;
  }
}

// Real Hessenberg reduction + Francis double-shift QR (real arithmetic), then
// the 2 x 2 blocks are triangularised: A = Z T Z^H with T upper triangular.
bool complex_schur(const std::vector<double>& A, int n, CMat& T, CMat& Z) {
  std::vector<double> H, Zr;
  if (!real_schur(A, n, H, Zr)) return false;
  complexify_schur(H, Zr, n, T, Z);
  return true;
}

bool complex_schur_c(const CMat& A, CMat& T, CMat& Z) {
  const int n = A.n;
  T = A;
  Z = CMat(n);
  for (int i = 0; i < n; ++i) Z(i, i) = 1.0;
  // Householder reduction to upper Hessenberg form: T <- H T H^H, Z <- Z H^H
  std::vector<cplx> v(n);
  for (int k = 0; k + 2 < n; ++k) {
    double xn2 = 0.0;
    for (int i = k + 1; i < n; ++i) xn2 += std::norm(T(i, k));
    if (xn2 == 0.0) continue;
    const double xn = std::sqrt(xn2);
    const cplx x0 = T(k + 1, k);
    const cplx ph = std::abs(x0) > 0.0 ? x0 / std::abs(x0) : cplx(1.0);
    const cplx alpha = -ph * xn;
    for (int i = k + 1; i < n; ++i) v[i] = T(i, k);
    v[k + 1] -= alpha;
    double vn2 = 0.0;
    for (int i = k + 1; i < n; ++i) vn2 += std::norm(v[i]);
    if (vn2 == 0.0) continue;
    const double tau = 2.0 / vn2;
    for (int j = k; j < n; ++j) {  // left: rows k+1.. of columns k..n-1
      cplx w = 0.0;
      for (int i = k + 1; i < n; ++i) w += std::conj(v[i]) * T(i, j);
      w *= tau;
      for (int i = k + 1; i < n; ++i) T(i, j) -= v[i] * w;
    }
    for (CMat* M : {&T, &Z}) {  // right: columns k+1.. (all rows)
      for (int i = 0; i < n; ++i) {
        cplx w = 0.0;
        for (int j = k + 1; j < n; ++j) w += (*M)(i, j) * v[j];
        w *= tau;
        for (int j = k + 1; j < n; ++j) (*M)(i, j) -= w * std::conj(v[j]);
      }
    }
    for (int i = k + 2; i < n; ++i) T(i, k) = 0.0;
  }
  // single-shift QR with Wilkinson shifts (complex Givens), deflation at
  // eps (|t_{l-1,l-1}| + |t_{l,l}|), an exceptional shift every 10 iterations
  const double eps = std::numeric_limits<double>::epsilon();
  int hi = n - 1, its = 0, total = 0;
  while (hi > 0) {
    int l = hi;
    for (; l > 0; --l)
      if (std::abs(T(l, l - 1)) <= eps * (std::abs(T(l - 1, l - 1)) + std::abs(T(l, l)))) {
        T(l, l - 1) = 0.0;
        break;
      }
    if (l == hi) {
      --hi;
      its = 0;
      continue;
    }
    if (++total > 30 * n) return false;
    ++its;
    cplx mu;
    const cplx a = T(hi - 1, hi - 1), b = T(hi - 1, hi), c = T(hi, hi - 1), d = T(hi, hi);
    if (its % 10 == 0) {
      mu = d + std::abs(c);
    } else {
      const cplx tr2 = 0.5 * (a + d), dsc = std::sqrt(0.25 * (a - d) * (a - d) + b * c);
      mu = std::abs(tr2 + dsc - d) < std::abs(tr2 - dsc - d) ? tr2 + dsc : tr2 - dsc;
    }
    for (int k = l; k < hi; ++k) {
      double cs;
      cplx sn;
      if (k == l)
        givens(T(l, l) - mu, T(l + 1, l), cs, sn);
      else
        givens(T(k, k - 1), T(k + 1, k - 1), cs, sn);
      rot_rows(T, k, k == l ? l : k - 1, n, cs, sn);
      if (k > l) T(k + 1, k - 1) = 0.0;
      rot_cols(T, k, 0, std::min(k + 3, hi + 1), cs, sn);
      rot_cols(Z, k, 0, n, cs, sn);
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

namespace {

// 3-element Householder reflector I - tau v v^T with v[piv] = 1 that maps u
// onto a multiple of e_piv (u is overwritten by v).
double house3(double* u, int piv) {
  const int a = piv == 0 ? 1 : 0, b = piv == 2 ? 1 : 2;
  const double xn = std::hypot(u[a], u[b]);
  if (xn == 0.0) {
    u[a] = u[b] = 0.0;
    u[piv] = 1.0;
    return 0.0;
  }
  const double alpha = u[piv];
  const double beta = -std::copysign(std::hypot(alpha, xn), alpha);
  const double sc = 1.0 / (alpha - beta);
  u[a] *= sc;
  u[b] *= sc;
  u[piv] = 1.0;
  return (beta - alpha) / beta;
}

// M[r..r+2, c0..c1) <- (I - tau v v^T) M[r..r+2, c0..c1)   (column-major, ld)
void refl3_left(double* M, int ld, int r, int c0, int c1, const double* v, double tau) {
  if (tau == 0.0) return;
  for (int c = c0; c < c1; ++c) {
    double* x = M + r + static_cast<size_t>(c) * ld;
    const double s = tau * (v[0] * x[0] + v[1] * x[1] + v[2] * x[2]);
    x[0] -= s * v[0];
    x[1] -= s * v[1];
    x[2] -= s * v[2];
  }
}

// M[r0..r1, c..c+2] <- M[r0..r1, c..c+2] (I - tau v v^T)
void refl3_right(double* M, int ld, int c, int r0, int r1, const double* v, double tau) {
  if (tau == 0.0) return;
  double* x0 = M + static_cast<size_t>(c) * ld;
  double* x1 = x0 + ld;
  double* x2 = x1 + ld;
  const double t0 = tau * v[0], t1 = tau * v[1], t2 = tau * v[2];
  for (int i = r0; i < r1; ++i) {
    const double s = v[0] * x0[i] + v[1] * x1[i] + v[2] * x2[i];
    x0[i] -= s * t0;
    x1[i] -= s * t1;
    x2[i] -= s * t2;
  }
}

// TL X - X TR = B for X (n1 x n2, n1, n2 <= 2), all column-major with the
// given leading dimensions: the n1 n2 Kronecker system by Gaussian elimination
// with complete pivoting, tiny pivots lifted to smin.
void small_sylvester(const double* TL, int ldl, const double* TR, int ldr, const double* B, int ldb, int n1, int n2,
                     double* X) {
  const int m = n1 * n2;
  double K[4][4] = {}, b[4];
  double kmax = 0.0;
  for (int j = 0; j < n2; ++j)
    for (int i = 0; i < n1; ++i) {
      const int row = i + j * n1;
      b[row] = B[i + j * ldb];
      for (int l = 0; l < n2; ++l)
        for (int k = 0; k < n1; ++k) {
          double v = 0.0;
          if (j == l) v += TL[i + k * ldl];
          if (i == k) v -= TR[l + j * ldr];
          K[row][k + l * n1] = v;
          kmax = std::max(kmax, std::fabs(v));
        }
    }
  const double smin = std::max(8.0 * std::numeric_limits<double>::epsilon() * kmax, 1e-290);
  int cperm[4] = {0, 1, 2, 3};
  for (int c = 0; c < m; ++c) {
    int pr = c, pc = c;
    double best = -1.0;
    for (int i = c; i < m; ++i)
      for (int j = c; j < m; ++j)
        if (std::fabs(K[i][j]) > best) best = std::fabs(K[i][j]), pr = i, pc = j;
    if (pr != c) {
      for (int j = 0; j < m; ++j) std::swap(K[pr][j], K[c][j]);
      std::swap(b[pr], b[c]);
    }
    if (pc != c) {
      for (int i = 0; i < m; ++i) std::swap(K[i][pc], K[i][c]);
      std::swap(cperm[pc], cperm[c]);
    }
    if (std::fabs(K[c][c]) < smin) K[c][c] = smin;
    for (int i = c + 1; i < m; ++i) {
      const double f = K[i][c] / K[c][c];
      for (int j = c; j < m; ++j) K[i][j] -= f * K[c][j];
      b[i] -= f * b[c];
    }
  }
  double x[4];
  for (int i = m - 1; i >= 0; --i) {
    double v = b[i];
    for (int j = i + 1; j < m; ++j) v -= K[i][j] * x[j];
    x[i] = v / K[i][i];
  }
  for (int i = 0; i < m; ++i) X[cperm[i]] = x[i];
}

// Swap the adjacent diagonal blocks T11 (n1 x n1, at j1) and T22 (n2 x n2) of
// the real Schur form by an orthogonal similarity, updating Z (the direct
// swapping method of Bai & Demmel, 1993: the Sylvester solution X of
// T11 X - X T22 = T12 spans the invariant subspace [-X; I] of T22, whose
// QR factor moves it up). Returns false (nothing changed) when the swapped
// form would not be block triangular to working accuracy.
bool swap_blocks(std::vector<double>& Tv, std::vector<double>& Zv, int n, int j1, int n1, int n2) {
  double* T = Tv.data();
  double* Z = Zv.data();
  auto t = [&](int i, int j) -> double& { return T[i + static_cast<size_t>(j) * n]; };
  if (n1 == 1 && n2 == 1) {
    const int j2 = j1 + 1;
    const double t11 = t(j1, j1), t22 = t(j2, j2);
    const double f = t(j1, j2), g = t22 - t11;
    const double r = std::hypot(f, g);
    if (r == 0.0) return true;  // equal eigenvalues, t12 = 0: nothing to move
    const double cs = f / r, sn = g / r;
    for (int j = j2 + 1; j < n; ++j) {
      const double x = t(j1, j), y = t(j2, j);
      t(j1, j) = cs * x + sn * y;
      t(j2, j) = cs * y - sn * x;
    }
    auto cols = [&](double* M, int rows) {
      double* c0 = M + static_cast<size_t>(j1) * n;
      double* c1 = c0 + n;
      for (int i = 0; i < rows; ++i) {
        const double x = c0[i], y = c1[i];
        c0[i] = cs * x + sn * y;
        c1[i] = cs * y - sn * x;
      }
    };
    cols(T, j1);
    cols(Z, n);
    t(j1, j1) = t22;
    t(j2, j2) = t11;
    return true;
  }
  const int nd = n1 + n2;
  double D[16];
  double dnorm = 0.0;
  for (int j = 0; j < nd; ++j)
    for (int i = 0; i < nd; ++i) {
      D[i + 4 * j] = t(j1 + i, j1 + j);
      dnorm = std::max(dnorm, std::fabs(D[i + 4 * j]));
    }
  const double thresh = std::max(10.0 * std::numeric_limits<double>::epsilon() * dnorm, 1e-290);
  double X[4];
  small_sylvester(D, 4, D + n1 + 4 * n1, 4, D + 4 * n1, 4, n1, n2, X);
  if (n1 == 1) {  // n2 = 2: reflector mapping (1, X11, X12) onto e_3
    double v[3] = {1.0, X[0], X[1]};
    const double tau = house3(v, 2);
    const double t11 = t(j1, j1);
    refl3_left(D, 4, 0, 0, 3, v, tau);
    refl3_right(D, 4, 0, 0, 3, v, tau);
    if (std::max({std::fabs(D[2]), std::fabs(D[2 + 4]), std::fabs(D[2 + 8] - t11)}) > thresh) return false;
    refl3_left(T, n, j1, j1, n, v, tau);
    refl3_right(T, n, j1, 0, j1 + 2, v, tau);
    refl3_right(Z, n, j1, 0, n, v, tau);
    t(j1 + 2, j1) = 0.0;
    t(j1 + 2, j1 + 1) = 0.0;
    t(j1 + 2, j1 + 2) = t11;
    return true;
  }
  if (n2 == 1) {  // n1 = 2: reflector mapping (-X11, -X21, 1) onto e_1
    double v[3] = {-X[0], -X[1], 1.0};
    const double tau = house3(v, 0);
    const double t33 = t(j1 + 2, j1 + 2);
    refl3_left(D, 4, 0, 0, 3, v, tau);
    refl3_right(D, 4, 0, 0, 3, v, tau);
    if (std::max({std::fabs(D[1]), std::fabs(D[2]), std::fabs(D[0] - t33)}) > thresh) return false;
    refl3_right(T, n, j1, 0, j1 + 3, v, tau);
    refl3_left(T, n, j1, j1 + 1, n, v, tau);
    refl3_right(Z, n, j1, 0, n, v, tau);
    t(j1, j1) = t33;
    t(j1 + 1, j1) = 0.0;
    t(j1 + 2, j1) = 0.0;
    return true;
  }
  // n1 = n2 = 2: two reflectors triangularise [-X; I]
  double v1[3] = {-X[0], -X[1], 1.0};
  const double tau1 = house3(v1, 0);
  const double tmp = -tau1 * (X[2] + v1[1] * X[3]);
  double v2[3] = {-tmp * v1[1] - X[3], -tmp * v1[2], 1.0};
  const double tau2 = house3(v2, 0);
  refl3_left(D, 4, 0, 0, 4, v1, tau1);
  refl3_right(D, 4, 0, 0, 4, v1, tau1);
  refl3_left(D, 4, 1, 0, 4, v2, tau2);
  refl3_right(D, 4, 1, 0, 4, v2, tau2);
  if (std::max({std::fabs(D[2]), std::fabs(D[2 + 4]), std::fabs(D[3]), std::fabs(D[3 + 4])}) > thresh) return false;
  refl3_left(T, n, j1, j1, n, v1, tau1);
  refl3_right(T, n, j1, 0, j1 + 4, v1, tau1);
  refl3_left(T, n, j1 + 1, j1, n, v2, tau2);
  refl3_right(T, n, j1 + 1, 0, j1 + 4, v2, tau2);
  refl3_right(Z, n, j1, 0, n, v1, tau1);
  refl3_right(Z, n, j1 + 1, 0, n, v2, tau2);
  t(j1 + 2, j1) = t(j1 + 2, j1 + 1) = t(j1 + 3, j1) = t(j1 + 3, j1 + 1) = 0.0;
  return true;
}

}  // namespace

int real_schur_reorder(std::vector<double>& T, std::vector<double>& Z, int n, std::vector<int>& sel) {
  auto sub = [&](int k) { return T[(k + 1) + static_cast<size_t>(k) * n]; };  // T(k+1, k)
  for (int k = 0; k + 1 < n; ++k)
    if (sub(k) != 0.0) {
      const int s = sel[k] || sel[k + 1];
      sel[k] = sel[k + 1] = s;
      ++k;
    }
  auto bsize = [&](int k) { return k + 1 < n && sub(k) != 0.0 ? 2 : 1; };
  int ks = 0;
  while (true) {
    int k = ks;
    while (k < n && !sel[k]) k += bsize(k);
    if (k >= n) break;
    int nb = bsize(k), here = k;
    while (here > ks) {
      const int nprev = here - 2 >= ks && sub(here - 2) != 0.0 ? 2 : 1;
      if (!swap_blocks(T, Z, n, here - nprev, nprev, nb)) return -1;
      std::rotate(sel.begin() + here - nprev, sel.begin() + here, sel.begin() + here + nb);
      here -= nprev;
      nb = bsize(here);
    }
    ks += bsize(ks);
  }
  return ks;
}

CMat triangular_eigvecs(const CMat& T) {
  const int n = T.n;
  CMat Y(n);
  double tnorm = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i <= j; ++i) tnorm = std::max(tnorm, std::abs(T(i, j)));
  const double smin = std::max(tnorm * std::numeric_limits<double>::epsilon(), 1e-300);
#pragma omp parallel for schedule(dynamic, 8) num_threads(host_threads()) if (n >= 96)
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
  // Column-pivoted Gram-Schmidt over the 2p candidates {Re z_j, Im z_j}: the
  // candidate of largest remaining norm is taken, re-orthogonalised once more
  // against the basis (every candidate is deflated against each new basis
  // vector as it is accepted, so with the extra pass this is CGS2), and the
  // remaining norms are downdated (recomputed once they lost 90% of their
  // last exact value).
  const int n = Z.n, nc = 2 * p;
  std::vector<double> C(static_cast<size_t>(n) * nc);
  for (int j = 0; j < p; ++j)
    for (int i = 0; i < n; ++i) {
      C[i + static_cast<size_t>(2 * j) * n] = Z(i, j).real();
      C[i + static_cast<size_t>(2 * j + 1) * n] = Z(i, j).imag();
    }
  auto col = [&](int j) { return C.data() + static_cast<size_t>(j) * n; };
  auto nrm2 = [&](const double* x) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += x[i] * x[i];
    return s;
  };
  Q.assign(static_cast<size_t>(n) * p, 0.0);
  std::vector<char> used(nc, 0);
  std::vector<double> nrm(nc), nrm_ref(nc);
  double maxn0 = 0.0;
  for (int j = 0; j < nc; ++j) {
    nrm[j] = nrm_ref[j] = nrm2(col(j));
    maxn0 = std::max(maxn0, std::sqrt(nrm[j]));
  }
  std::vector<double> q(n);
  int rank = 0;
  while (rank < p) {
    int best = -1;
    double bn = 0.0;
    for (int j = 0; j < nc; ++j)
      if (!used[j] && nrm[j] > bn) bn = nrm[j], best = j;
    if (best < 0 || std::sqrt(bn) <= 1e-10 * maxn0) break;
    used[best] = 1;
    std::copy(col(best), col(best) + n, q.begin());
    for (int r = 0; r < rank; ++r) {  // second Gram-Schmidt pass
      const double* qr = Q.data() + static_cast<size_t>(r) * n;
      double d = 0;
      for (int i = 0; i < n; ++i) d += qr[i] * q[i];
      for (int i = 0; i < n; ++i) q[i] -= d * qr[i];
    }
    double s = std::sqrt(nrm2(q.data()));
    if (s <= 1e-12 * maxn0) continue;
    double* qn = Q.data() + static_cast<size_t>(rank) * n;
    for (int i = 0; i < n; ++i) qn[i] = q[i] / s;
    ++rank;
    // deflate the remaining candidates, downdate their norms
#pragma omp parallel for schedule(static) num_threads(host_threads()) if (static_cast<int64_t>(n) * nc > 20000)
    for (int j = 0; j < nc; ++j) {
      if (used[j]) continue;
      double* cj = col(j);
      double d = 0;
      for (int i = 0; i < n; ++i) d += qn[i] * cj[i];
      for (int i = 0; i < n; ++i) cj[i] -= d * qn[i];
      nrm[j] -= d * d;
      if (nrm[j] <= 0.1 * nrm_ref[j]) nrm[j] = nrm_ref[j] = nrm2(cj);
    }
  }
  return rank;
}

}  // namespace rqb
