// SPDX-License-Identifier: Apache-2.0
// Small dense eigen-kernels for the m x m projected problem (m <= 512) of the
// Krylov-Schur driver: ritz_extract / krylov_schur_restart.
// Complex Schur form of the real projected matrix (Householder Hessenberg +
// single-shift QR with Wilkinson shifts), adjacent Givens swaps to reorder it,
// triangular eigenvectors, and a pivoted Gram-Schmidt that turns a
// conjugation-closed set of complex Schur vectors into a real orthonormal
// basis, so every N-sized vector on the device stays real.
#pragma once

#include <complex>
#include <vector>

namespace rqb {

using cplx = std::complex<double>;

// column-major n x n helpers
struct CMat {
  int n = 0;
  std::vector<cplx> a;
  explicit CMat(int n_ = 0) : n(n_), a(static_cast<size_t>(n_) * n_) {}
  cplx& operator()(int i, int j) { return a[i + static_cast<size_t>(j) * n]; }
  cplx operator()(int i, int j) const { return a[i + static_cast<size_t>(j) * n]; }
};

// A = Z T Z^H with T upper triangular. Returns false if QR did not converge
// within 30 n iterations per eigenvalue.
bool complex_schur(const std::vector<double>& A, int n, CMat& T, CMat& Z);

// A = Z T Z^H for a complex A (Householder Hessenberg + single-shift complex
// QR with Wilkinson shifts). Returns false past 30 n iterations.
bool complex_schur_c(const CMat& A, CMat& T, CMat& Z);

// Move the selected diagonal entries of T to the leading positions (stable
// order), updating Z. sel is permuted alongside.
void schur_reorder(CMat& T, CMat& Z, std::vector<int>& sel);

// Eigenvectors of the upper-triangular T (columns), unit 2-norm.
CMat triangular_eigvecs(const CMat& T);

// Real orthonormal basis (n x p, column-major) of span{Re Z[:, :p], Im Z[:, :p]}
// of numerical rank p. Returns the rank found.
int real_basis(const CMat& Z, int p, std::vector<double>& Q);

}  // namespace rqb
