// SPDX-License-Identifier: Apache-2.0
// Complex Krylov-Schur for complex pencils / complex shifts:
// the device engine (cuda/zkrylov.cu) and the host driver (host/zeigs.cpp).
#pragma once

#include <complex>
#include <cstdint>
#include <memory>
#include <vector>

#include "../engine.hpp"

namespace rqb {

// Shift-invert operator of the linearised pencil with complex K, C, M (values
// interleaved {re, im} on one pattern) and a complex shift s; Q(s) factored as
// its real-equivalent 2n system. Vectors: [v_u | v_l], n complex each.
struct ZOperatorEngine {
  int64_t n = 0, nnz = 0;
  double s_re = 0.0, s_im = 0.0;
  std::unique_ptr<FactorEngine> fac;
  DeviceBuffer d_rowptr, d_col, d_K, d_C, d_M, d_t, d_part, d_res;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  ZOperatorEngine(int64_t n, const int64_t* rowptr, const int32_t* col, const double* K, const double* C,
                  const double* M, const Symbolic& s2, double sr, double si, const std::vector<int64_t>& rp2,
                  const std::vector<int32_t>& col2, const std::vector<double>& q2);
  void spmv(int which, const double* x, double* y);  // y = A x, A in {0 K, 1 C, 2 M}, n complex
  void apply(const double* v, double* r);            // r = L(s)^{-1} B v
  void bvec(const double* r, double* w);             // w = [r_u; M r_l]
  // h[i] = V_i^H w (complex), i < k, vectors of 2n complex at stride ldv doubles
  void gemv_t(const double* V, int k, int64_t ldv, const double* w, double* h);
  void gemv_n(const double* V, int k, int64_t ldv, const double* h, double* r);  // r -= V h
  // beta = sqrt(Re r^H w); v = r / beta, bv = w / beta
  void bnorm_normalize(const double* r, const double* w, double* beta_out, double* v, double* bv);
  // X[:, c] = V Q[:, c] over len complex entries (Q: k x nc complex, column-major, ldq)
  void combine(const double* V, int k, int64_t ldv, int64_t len, const double* Q, int ldq, int nc, double* X,
               int64_t ldx);
  // out[2c] = ||K u + lam C u + lam^2 M u||^2, out[2c+1] = ||u||^2, u at X + c ldx (n complex)
  void residuals(const double* X, int64_t ldx, int nc, const double* lam_host, double* out_host);
};

struct ZEigsOptions {
  int nev = 10, m = 0;
  double tol = 1e-10;
  uint64_t seed = 0;
  int max_restarts = 100;
  int want_vectors = 0;
};

struct ZEigsResult {
  bool converged = false;
  int nconv = 0, cycles = 0;
  std::vector<std::complex<double>> lambda;
  std::vector<double> resid;
  std::vector<double> vec;  // n x nev complex (interleaved), unit 2-norm
  int64_t launches = 0;
};

ZEigsResult solve_quadratic_complex(ZOperatorEngine& E, const ZEigsOptions& o, const double norms1[3]);

}  // namespace rqb
