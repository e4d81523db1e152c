// SPDX-License-Identifier: Apache-2.0
// solve_generalized_hermitian: shift-invert Lanczos with
// thick restarts on the device (host/lanczos.cpp).
#pragma once

#include <cstdint>
#include <vector>

namespace rqb {

struct GhEngine;

struct GhOptions {
  int nev = 10;
  int m = 0;  // <= 0: max(2 nev, nev + 20)
  double tol = 1e-10;
  uint64_t seed = 0;
  int max_restarts = 100;
  double est_factor = 1e3;
  int want_vectors = 0;
};

struct GhResult {
  bool converged = false;
  int nconv = 0, cycles = 0, restarts = 0;
  std::vector<double> lam, resid, vec;  // vec: n x nev column-major, unit 2-norm
  double lanczos_defect = 0.0;  // max |v_i^T B S v_j|, i < j-1 (three-term structure), / ||T||
  double sym_defect = 0.0;      // max |v_{j-1}^T B S v_j - beta_{j-1}| / ||T|| (B-self-adjointness)
  int64_t launches = 0;
};

// Symmetric eigen-decomposition (cyclic Jacobi), column-major.
void sym_eig_jacobi(std::vector<double> A, int n, std::vector<double>& w, std::vector<double>& Z);

GhResult solve_generalized_hermitian_device(GhEngine& E, const GhOptions& o, double normA1, double normB1);

}  // namespace rqb
