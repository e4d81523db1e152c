// SPDX-License-Identifier: Apache-2.0
// solve_generalized_hermitian (Alg. 1 + Remark 3):
// nev eigenpairs of A u = lambda B u nearest a real shift s, A symmetric, B
// symmetric positive definite (the non-conductive Maxwell problem of §6.4.1,
// Remark 2: K u = omega^2 M u). Shift-invert Lanczos on S = (A - s B)^{-1} B,
// which is B-self-adjoint: with a B-orthonormal basis the projected matrix is
// the symmetric tridiagonal T_m (Remark 3: orthogonalization "only performed
// against the last two basis vectors"; here every step also runs one full
// CGS2 reorthogonalization pass, the SPEC's "selective reorthogonalization
// engaged" taken always, so ||V^T B V - I|| stays at rounding level; its
// coefficients are not added to T, whose entries come from the three-term
// recurrence alone). Thick restart (Krylov-Schur for symmetric T): keep the
// p Ritz vectors nearest the shift, T becomes diag(theta_p) bordered by the
// residual row b = beta_m Y[m-1, :p] (an arrowhead), the next Lanczos step
// couples to all kept vectors through b. Ritz values are real; lambda = s +
// 1/theta. Convergence on the explicit residual
//   ||A u - lambda B u|| / ((||A||_1 + |lambda| ||B||_1) ||u||) <= tol.
// Every N-sized vector lives on the device (GhEngine, cuda/krylov.cu).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "../engine.hpp"
#include "lanczos.hpp"

namespace rqb {

// Cyclic Jacobi eigen-decomposition of the symmetric n x n A (column-major):
// w eigenvalues, Z orthonormal eigenvectors (columns). High relative accuracy;
// O(n^3) per sweep, fine for the m <= a few hundred projected matrices here.
void sym_eig_jacobi(std::vector<double> A, int n, std::vector<double>& w, std::vector<double>& Z) {
  Z.assign(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i) Z[i + static_cast<size_t>(i) * n] = 1.0;
  auto a = [&](int i, int j) -> double& { return A[i + static_cast<size_t>(j) * n]; };
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        tot += a(i, j) * a(i, j);
        if (i != j) off += a(i, j) * a(i, j);
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = a(p, q);
        if (std::fabs(apq) <= 1e-300) continue;
        const double app = a(p, p), aqq = a(q, q);
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {  // columns p, q
          const double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {  // rows p, q
          const double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
        a(p, q) = a(q, p) = 0.0;
        for (int k = 0; k < n; ++k) {
          double* zp = &Z[k + static_cast<size_t>(p) * n];
          double* zq = &Z[k + static_cast<size_t>(q) * n];
          const double x = *zp, y = *zq;
          *zp = c * x - s * y;
          *zq = s * x + c * y;
        }
      }
  }
  w.resize(n);
  for (int i = 0; i < n; ++i) w[i] = a(i, i);
}

GhResult solve_generalized_hermitian_device(GhEngine& E, const GhOptions& o, double normA1, double normB1) {
  const int64_t n = E.n;
  const int nev = o.nev;
  const int m = o.m > 0 ? o.m : std::max(2 * nev, nev + 20);  // SPEC.md:489 default sizing
  if (nev < 1) fail(errc::config, "nev must be positive");
  if (m <= nev && m < n) fail(errc::config, "Krylov dimension m must exceed nev (or span the whole space)");
  if (m > 512) fail(errc::config, "Krylov dimension above 512");
  if (m > n) fail(errc::config, "Krylov dimension must not exceed N");
  if (!(o.tol > 0)) fail(errc::config, "tolerance must be positive");
  const int keep_target = nev + std::min(20, m - nev - 1);
  const double s = E.shift;
  cudaStream_t st = E.stream;
  const int64_t launches0 = E.launches;
  GhResult res;

  DeviceBuffer dV, dBV, dV2, dBV2, dR, dHa, dHb, dBeta, dQ, dX;
  dV.alloc(sizeof(double) * (m + 1) * n);
  dBV.alloc(sizeof(double) * (m + 1) * n);
  dV2.alloc(sizeof(double) * (m + 1) * n);
  dBV2.alloc(sizeof(double) * (m + 1) * n);
  dR.alloc(sizeof(double) * n);
  dHa.alloc(sizeof(double) * (m + 1) * (m + 1));
  dHb.alloc(sizeof(double) * (m + 1) * (m + 1));
  dBeta.alloc(sizeof(double) * (m + 1));
  dQ.alloc(sizeof(double) * (m + 1) * (m + 1));
  dX.alloc(sizeof(double) * n * (m + 1));
  double* V = dV.as<double>();
  double* BV = dBV.as<double>();
  double* V2 = dV2.as<double>();
  double* BV2 = dBV2.as<double>();
  double* r = dR.as<double>();

  auto fresh = [&](uint64_t seed, int nlock) {
    std::vector<double> v(n);
    uint64_t x = seed;
    for (int64_t i = 0; i < n; ++i) v[i] = splitmix_uniform(x);
    cuda_check(cudaMemcpyAsync(r, v.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st), "H2D v0");
    for (int pass = 0; pass < 2 && nlock > 0; ++pass) {
      E.gemv_t(BV, nlock, r, dHa.as<double>());
      E.gemv_n(V, nlock, dHa.as<double>(), r);
    }
    E.bnorm_normalize(r, dBeta.as<double>() + m, V + static_cast<int64_t>(nlock) * n,
                      BV + static_cast<int64_t>(nlock) * n);
    cuda_check(cudaStreamSynchronize(st), "sync");
  };

  // T: symmetric (m+1) x (m+1), column-major; diagonal alpha, off-diagonal beta,
  // plus the arrowhead coupling of the kept block after a restart
  std::vector<double> T(static_cast<size_t>(m + 1) * (m + 1), 0.0);
  auto Tc = [&](int i, int j) -> double& { return T[i + static_cast<size_t>(j) * (m + 1)]; };
  std::vector<double> ha(static_cast<size_t>(m + 1) * (m + 1)), hb(ha.size()), betas(m + 1);
  fresh(o.seed, 0);
  int k = 0;
  std::vector<double> final_lam, final_res, final_vec;
  while (res.cycles < o.max_restarts) {
    ++res.cycles;
    int mm = m;  // steps actually taken (breakdown: invariant subspace)
    for (int j = k; j < m; ++j) {
      double* hA = dHa.as<double>() + static_cast<int64_t>(j) * (m + 1);
      double* hB = dHb.as<double>() + static_cast<int64_t>(j) * (m + 1);
      E.apply(V + static_cast<int64_t>(j) * n, r);
      E.gemv_t(BV, j + 1, r, hA);
      E.gemv_n(V, j + 1, hA, r);
      E.gemv_t(BV, j + 1, r, hB);
      E.gemv_n(V, j + 1, hB, r);
      E.bnorm_normalize(r, dBeta.as<double>() + j, V + static_cast<int64_t>(j + 1) * n,
                        BV + static_cast<int64_t>(j + 1) * n);
    }
    cuda_check(cudaMemcpyAsync(ha.data(), dHa.p, sizeof(double) * ha.size(), cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaMemcpyAsync(hb.data(), dHb.p, sizeof(double) * hb.size(), cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaMemcpyAsync(betas.data(), dBeta.p, sizeof(double) * (m + 1), cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
    E.fac->check_sweeps();
    double tnorm = 0.0, ldef = 0.0, sdef = 0.0;
    for (int j = k; j < m; ++j) {
      const double* a = &ha[static_cast<size_t>(j) * (m + 1)];
      const double* b = &hb[static_cast<size_t>(j) * (m + 1)];
      const double alpha = a[j] + b[j];
      Tc(j, j) = alpha;
      tnorm = std::max(tnorm, std::fabs(alpha) + betas[j]);
      // Lanczos structure: projections on v_i, i < j-1 (other than the kept
      // block's arrowhead on the first step after a restart) vanish up to
      // rounding; the recurrence's T ignores them (defect recorded)
      for (int i = 0; i + 1 < j; ++i) {
        if (j == k && i < k) continue;
        ldef = std::max(ldef, std::fabs(a[i] + b[i]));
      }
      if (j > k) {  // symmetry of the computed projection: h_{j-1,j} vs beta_{j-1}
        sdef = std::max(sdef, std::fabs(a[j - 1] + b[j - 1] - betas[j - 1]));
      }
      Tc(j + 1, j) = Tc(j, j + 1) = betas[j];
      if (betas[j] <= 1e-14 * std::max(1.0, tnorm)) {  // invariant subspace: every Ritz pair exact
        mm = j + 1;
        break;
      }
    }
    res.lanczos_defect = std::max(res.lanczos_defect, ldef / std::max(tnorm, 1e-300));
    res.sym_defect = std::max(res.sym_defect, sdef / std::max(tnorm, 1e-300));
    // ---- Ritz pairs of T_mm (real: symmetric) ----
    std::vector<double> Tm(static_cast<size_t>(mm) * mm);
    for (int j = 0; j < mm; ++j)
      for (int i = 0; i < mm; ++i) Tm[i + static_cast<size_t>(j) * mm] = Tc(i, j);
    std::vector<double> th, Y;
    sym_eig_jacobi(Tm, mm, th, Y);
    const double beta_m = mm < m ? 0.0 : betas[m - 1];
    std::vector<int> order(mm);
    std::iota(order.begin(), order.end(), 0);
    auto lam_of = [&](int i) { return s + 1.0 / th[i]; };
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return std::fabs(lam_of(a) - s) < std::fabs(lam_of(b) - s);
    });
    const int nw = std::min(nev, mm);
    double est_worst = 0.0;
    for (int c = 0; c < nw; ++c) {
      const int i = order[c];
      est_worst = std::max(est_worst, std::fabs(beta_m * Y[(mm - 1) + static_cast<size_t>(i) * mm]) /
                                          std::max(std::fabs(th[i]), 1e-300));
    }
    bool all = false;
    if (est_worst <= o.est_factor * o.tol || mm < m) {
      // Ritz vectors X = V_mm Y[:, order[0..nw)] and their explicit residuals
      std::vector<double> Yc(static_cast<size_t>(mm) * nw);
      for (int c = 0; c < nw; ++c)
        std::memcpy(&Yc[static_cast<size_t>(c) * mm], &Y[static_cast<size_t>(order[c]) * mm], sizeof(double) * mm);
      cuda_check(cudaMemcpyAsync(dQ.p, Yc.data(), sizeof(double) * Yc.size(), cudaMemcpyHostToDevice, st), "H2D");
      vq_gemm(V, n, n, mm, dQ.as<double>(), mm, nw, dX.as<double>(), n, false, st);
      ++E.launches;
      std::vector<double> lam(nw), rr(2 * nw);
      for (int c = 0; c < nw; ++c) lam[c] = lam_of(order[c]);
      E.residuals(dX.as<double>(), nw, lam.data(), rr.data());
      all = true;
      final_lam.assign(lam.begin(), lam.end());
      final_res.assign(nw, 1.0);
      for (int c = 0; c < nw; ++c) {
        const double den = (normA1 + std::fabs(lam[c]) * normB1) * std::sqrt(rr[2 * c + 1]);
        final_res[c] = den > 0 ? std::sqrt(rr[2 * c]) / den : 1.0;
        if (!(final_res[c] <= o.tol)) all = false;
      }
      if (all && o.want_vectors) {
        final_vec.resize(static_cast<size_t>(n) * nw);
        cuda_check(cudaMemcpyAsync(final_vec.data(), dX.p, sizeof(double) * final_vec.size(),
                                   cudaMemcpyDeviceToHost, st), "D2H x");
        cuda_check(cudaStreamSynchronize(st), "sync");
        for (int c = 0; c < nw; ++c) {  // unit 2-norm
          double nr = 0.0;
          for (int64_t i = 0; i < n; ++i) nr += final_vec[c * n + i] * final_vec[c * n + i];
          nr = std::sqrt(nr);
          for (int64_t i = 0; i < n; ++i) final_vec[c * n + i] /= nr;
        }
      }
    }
    if (all || mm < m) break;
    // ---- thick restart: keep the p nearest Ritz vectors; T = diag(theta_p) + arrow b ----
    const int p = std::min(keep_target, m - 1);
    std::vector<double> Qp(static_cast<size_t>(mm) * p);
    for (int c = 0; c < p; ++c)
      std::memcpy(&Qp[static_cast<size_t>(c) * mm], &Y[static_cast<size_t>(order[c]) * mm], sizeof(double) * mm);
    cuda_check(cudaMemcpyAsync(dQ.p, Qp.data(), sizeof(double) * Qp.size(), cudaMemcpyHostToDevice, st), "H2D Q");
    vq_gemm(V, n, n, mm, dQ.as<double>(), mm, p, V2, n, false, st);
    vq_gemm(BV, n, n, mm, dQ.as<double>(), mm, p, BV2, n, false, st);
    E.launches += 2;
    cuda_check(cudaMemcpyAsync(V2 + static_cast<int64_t>(p) * n, V + static_cast<int64_t>(mm) * n,
                               sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "D2D");
    cuda_check(cudaMemcpyAsync(BV2 + static_cast<int64_t>(p) * n, BV + static_cast<int64_t>(mm) * n,
                               sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "D2D");
    std::swap(V, V2);
    std::swap(BV, BV2);
    std::fill(T.begin(), T.end(), 0.0);
    for (int c = 0; c < p; ++c) {
      Tc(c, c) = th[order[c]];
      const double b = beta_m * Y[(mm - 1) + static_cast<size_t>(order[c]) * mm];
      Tc(p, c) = Tc(c, p) = b;
    }
    k = p;
    ++res.restarts;
  }
  E.fac->check_sweeps();
  res.lam = final_lam;
  res.resid = final_res;
  res.vec = std::move(final_vec);
  res.nconv = static_cast<int>(std::count_if(res.resid.begin(), res.resid.end(), [&](double x) { return x <= o.tol; }));
  res.converged = res.nconv >= std::min(nev, static_cast<int>(res.lam.size())) && !res.lam.empty();
  res.launches = E.launches - launches0;
  return res;
}

}  // namespace rqb
