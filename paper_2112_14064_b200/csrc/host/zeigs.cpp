// SPDX-License-Identifier: Apache-2.0
// Complex Krylov-Schur (SPEC.md:435-470 over complex scalars):
// the shift-invert operator of a complex pencil / complex shift
// (ZOperatorEngine), B-orthogonal CGS2 Arnoldi with conjugated projections,
// complex Schur form of H_m on the host (complex_schur_c), Ritz values lambda =
// s + 1/theta, explicit pencil residuals of the nev nearest once their
// estimates |beta_m e_m^H y| / |theta| pass 1e3 tol, restart keeping the keep =
// nev + min(20, m - nev - 1) nearest Schur directions (complex Schur vectors:
// no conjugation closure needed). Every N-sized vector lives on the device.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "dense.hpp"
#include "zeigs.hpp"

namespace rqb {

ZEigsResult solve_quadratic_complex(ZOperatorEngine& E, const ZEigsOptions& o, const double norms1[3]) {
  const int64_t n = E.n, ld = 4 * n;  // doubles per 2n complex Krylov vector
  const int nev = o.nev;
  const int m = o.m > 0 ? o.m : 2 * nev + 1;
  if (nev < 1) fail(errc::config, "nev must be positive");
  if (m <= nev) fail(errc::config, "Krylov dimension m must exceed nev");
  if (m > 512) fail(errc::config, "Krylov dimension above 512");
  if (m >= 2 * n) fail(errc::config, "Krylov dimension must be below 2N");
  const int keep = nev + std::min(20, m - nev - 1);
  const cplx s(E.s_re, E.s_im);
  cudaStream_t st = E.stream;
  const int64_t l0 = E.launches;
  DeviceBuffer dV, dBV, dV2, dBV2, dR, dW, dHa, dHb, dBeta, dQ, dX;
  dV.alloc(sizeof(double) * (m + 1) * ld);
  dBV.alloc(sizeof(double) * (m + 1) * ld);
  dV2.alloc(sizeof(double) * (m + 1) * ld);
  dBV2.alloc(sizeof(double) * (m + 1) * ld);
  dR.alloc(sizeof(double) * ld);
  dW.alloc(sizeof(double) * ld);
  dHa.alloc(sizeof(double) * 2 * (m + 1) * (m + 1));
  dHb.alloc(sizeof(double) * 2 * (m + 1) * (m + 1));
  dBeta.alloc(sizeof(double) * (m + 1));
  dQ.alloc(sizeof(double) * 2 * (m + 1) * (m + 1));
  dX.alloc(sizeof(double) * ld * std::max(nev, 1));
  double *V = dV.as<double>(), *BV = dBV.as<double>(), *V2 = dV2.as<double>(), *BV2 = dBV2.as<double>();
  double *r = dR.as<double>(), *w = dW.as<double>();
  auto fresh = [&](uint64_t seed, int nlock) {  // real uniform[-1,1] start (splitmix64), B-normalised
    std::vector<double> v(ld, 0.0);
    uint64_t x = seed;
    for (int64_t i = 0; i < 2 * n; ++i) v[2 * i] = splitmix_uniform(x);
    cuda_check(cudaMemcpyAsync(r, v.data(), sizeof(double) * ld, cudaMemcpyHostToDevice, st), "H2D v0");
    for (int pass = 0; pass < 2 && nlock > 0; ++pass) {
      E.gemv_t(BV, nlock, ld, r, dHa.as<double>());
      E.gemv_n(V, nlock, ld, dHa.as<double>(), r);
    }
    E.bvec(r, w);
    E.bnorm_normalize(r, w, dBeta.as<double>() + m, V + static_cast<int64_t>(nlock) * ld,
                      BV + static_cast<int64_t>(nlock) * ld);
    cuda_check(cudaStreamSynchronize(st), "sync");
  };
  CMat H(m + 1);  // (m+1) x (m+1), columns 0..m-1 used
  std::vector<double> ha(2 * static_cast<size_t>(m + 1) * (m + 1)), hb(ha.size()), betas(m + 1);
  fresh(o.seed, 0);
  int k = 0;
  ZEigsResult res;
  while (res.cycles < o.max_restarts) {
    ++res.cycles;
    for (int j = k; j < m; ++j) {
      double* hA = dHa.as<double>() + 2 * static_cast<int64_t>(j) * (m + 1);
      double* hB = dHb.as<double>() + 2 * static_cast<int64_t>(j) * (m + 1);
      E.apply(V + static_cast<int64_t>(j) * ld, r);
      E.gemv_t(BV, j + 1, ld, r, hA);  // h = (B V)^H r = V^H B r (B Hermitian)
      E.gemv_n(V, j + 1, ld, hA, r);
      E.gemv_t(BV, j + 1, ld, r, hB);
      E.gemv_n(V, j + 1, ld, hB, r);
      E.bvec(r, w);
      E.bnorm_normalize(r, w, dBeta.as<double>() + j, V + static_cast<int64_t>(j + 1) * ld,
                        BV + static_cast<int64_t>(j + 1) * ld);
    }
    cuda_check(cudaMemcpyAsync(ha.data(), dHa.p, sizeof(double) * ha.size(), cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaMemcpyAsync(hb.data(), dHb.p, sizeof(double) * hb.size(), cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaMemcpyAsync(betas.data(), dBeta.p, sizeof(double) * (m + 1), cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
    E.fac->check_sweeps();
    for (int j = k; j < m; ++j) {
      for (int i = 0; i <= j; ++i) {
        const size_t q = 2 * (i + static_cast<size_t>(j) * (m + 1));
        H(i, j) = cplx(ha[q] + hb[q], ha[q + 1] + hb[q + 1]);
      }
      H(j + 1, j) = betas[j];
    }
    CMat Hm(m);
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < m; ++i) Hm(i, j) = H(i, j);
    CMat T, Z;
    if (!complex_schur_c(Hm, T, Z)) fail(errc::solver, "complex Schur form did not converge");
    const CMat Y = triangular_eigvecs(T);
    std::vector<cplx> th(m), lam(m);
    std::vector<double> est(m);
    const double bm = H(m, m - 1).real();
    for (int i = 0; i < m; ++i) {
      th[i] = T(i, i);
      lam[i] = s + 1.0 / th[i];
      cplx yl = 0.0;
      for (int t = 0; t <= i; ++t) yl += Z(m - 1, t) * Y(t, i);
      est[i] = std::abs(bm * yl) / std::max(std::abs(th[i]), 1e-300);
    }
    std::vector<int> ord(m);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return std::abs(lam[a] - s) < std::abs(lam[b] - s); });
    bool all = true;
    for (int c = 0; c < nev; ++c) all = all && est[ord[c]] <= 1e3 * o.tol;
    if (all) {
      // Ritz vectors x_c = V_m y_c of the nev nearest, the pencil residual on the larger block
      std::vector<double> Yc(2 * static_cast<size_t>(m) * nev, 0.0), lamc(2 * nev), rr(2 * nev);
      for (int c = 0; c < nev; ++c) {
        const int i = ord[c];
        for (int row = 0; row < m; ++row) {
          cplx y = 0.0;
          for (int t = 0; t <= i; ++t) y += Z(row, t) * Y(t, i);
          Yc[2 * (row + static_cast<size_t>(c) * m)] = y.real();
          Yc[2 * (row + static_cast<size_t>(c) * m) + 1] = y.imag();
        }
        lamc[2 * c] = lam[i].real();
        lamc[2 * c + 1] = lam[i].imag();
      }
      cuda_check(cudaMemcpyAsync(dQ.p, Yc.data(), sizeof(double) * Yc.size(), cudaMemcpyHostToDevice, st), "H2D");
      E.combine(V, m, ld, 2 * n, dQ.as<double>(), m, nev, dX.as<double>(), ld);
      // residual per candidate on its block: |lambda| > 1 -> lower block (lambda u)
      std::vector<double> rup(2 * nev), rlo(2 * nev);
      E.residuals(dX.as<double>(), ld, nev, lamc.data(), rup.data());
      E.residuals(dX.as<double>() + 2 * n, ld, nev, lamc.data(), rlo.data());
      res.lambda.clear();
      res.resid.assign(nev, 1.0);
      std::vector<int> blk(nev, 0);
      for (int c = 0; c < nev; ++c) {
        const cplx lc = lam[ord[c]];
        const double al = std::abs(lc);
        blk[c] = al > 1.0 ? 1 : 0;
        const double* rv = blk[c] ? rlo.data() : rup.data();
        const double den = (norms1[0] + al * norms1[1] + al * al * norms1[2]) * std::sqrt(rv[2 * c + 1]);
        res.resid[c] = den > 0 ? std::sqrt(rv[2 * c]) / den : 1.0;
        res.lambda.push_back(lc);
        if (!(res.resid[c] <= o.tol)) all = false;
      }
      if (all) {
        if (o.want_vectors) {
          std::vector<double> X(ld * static_cast<size_t>(nev));
          cuda_check(cudaMemcpyAsync(X.data(), dX.p, sizeof(double) * X.size(), cudaMemcpyDeviceToHost, st), "D2H");
          cuda_check(cudaStreamSynchronize(st), "sync");
          res.vec.assign(2 * static_cast<size_t>(n) * nev, 0.0);
          for (int c = 0; c < nev; ++c) {
            const double* src = X.data() + static_cast<size_t>(c) * ld + (blk[c] ? 2 * n : 0);
            double nr = 0.0;
            for (int64_t e = 0; e < 2 * n; ++e) nr += src[e] * src[e];
            nr = std::sqrt(nr);
            for (int64_t e = 0; e < 2 * n; ++e) res.vec[static_cast<size_t>(c) * 2 * n + e] = src[e] / nr;
          }
        }
        res.converged = true;
        break;
      }
    }
    // restart: the keep nearest Schur directions lead; V <- V Z_p, H <- [T_p; beta_m Z(m-1, :p)]
    std::vector<int> sel(m, 0);
    for (int c = 0; c < std::min(keep, m - 1); ++c) sel[ord[c]] = 1;
    int p = 0;
    for (int v : sel) p += v;
    schur_reorder(T, Z, sel);
    std::vector<double> Zp(2 * static_cast<size_t>(m) * p);
    for (int c = 0; c < p; ++c)
      for (int row = 0; row < m; ++row) {
        Zp[2 * (row + static_cast<size_t>(c) * m)] = Z(row, c).real();
        Zp[2 * (row + static_cast<size_t>(c) * m) + 1] = Z(row, c).imag();
      }
    cuda_check(cudaMemcpyAsync(dQ.p, Zp.data(), sizeof(double) * Zp.size(), cudaMemcpyHostToDevice, st), "H2D Q");
    E.combine(V, m, ld, 2 * n, dQ.as<double>(), m, p, V2, ld);
    E.combine(BV, m, ld, 2 * n, dQ.as<double>(), m, p, BV2, ld);
    cuda_check(cudaMemcpyAsync(V2 + static_cast<int64_t>(p) * ld, V + static_cast<int64_t>(m) * ld,
                               sizeof(double) * ld, cudaMemcpyDeviceToDevice, st), "D2D");
    cuda_check(cudaMemcpyAsync(BV2 + static_cast<int64_t>(p) * ld, BV + static_cast<int64_t>(m) * ld,
                               sizeof(double) * ld, cudaMemcpyDeviceToDevice, st), "D2D");
    std::swap(V, V2);
    std::swap(BV, BV2);
    H = CMat(m + 1);
    for (int c = 0; c < p; ++c) {
      for (int i = 0; i <= c; ++i) H(i, c) = T(i, c);
      H(p, c) = bm * Z(m - 1, c);
    }
    k = p;
  }
  res.nconv = static_cast<int>(std::count_if(res.resid.begin(), res.resid.end(), [&](double x) { return x <= o.tol; }));
  res.launches = E.launches - l0;
  return res;
}

}  // namespace rqb
