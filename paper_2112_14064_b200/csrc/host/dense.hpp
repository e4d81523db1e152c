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

// The real Schur form behind complex_schur: A = Z T Z^T, T upper
// quasi-triangular (1 x 1 blocks and 2 x 2 blocks of complex-conjugate pairs),
// Z orthogonal, both n x n column-major.
bool real_schur(const std::vector<double>& A, int n, std::vector<double>& T, std::vector<double>& Z);

// The complex triangular form of a real Schur form (one complex rotation per
// 2 x 2 block; diagonal positions are kept: the pair of block k sits at k, k+1).
void complexify_schur(const std::vector<double>& T, const std::vector<double>& Z, int n, CMat& Tc, CMat& Zc);

// Move the selected blocks of the real Schur form (T, Z) to the leading
// positions (stable order) by adjacent block swaps; a 2 x 2 block is selected
// if either of its diagonal positions is (sel is closed over blocks and
// permuted alongside). Returns the order p of the leading selected part
// (T[:p, :p] quasi-triangular, Z[:, :p] an orthonormal real basis of its
// invariant subspace), or -1 if a swap was refused as inaccurate (T, Z are
// then partly reordered but still a valid Schur form).
int real_schur_reorder(std::vector<double>& T, std::vector<double>& Z, int n, std::vector<int>& sel);

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
