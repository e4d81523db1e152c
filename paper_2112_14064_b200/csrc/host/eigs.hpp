// SPDX-License-Identifier: Apache-2.0
#pragma once

#include <complex>
#include <cstdint>
#include <string>
#include <vector>

namespace rqb {

struct OperatorEngine;

// Four-category ledger + aux tallies (reference sparse.hpp:49-103). The GPU
// path computes in real FP64, so one multiply-add is 2 flops.
struct Ledger {
  int64_t n_fa = 0, n_fb = 0, n_mv = 0, n_vv = 0, n_check = 0, n_restart = 0;
  double macs_fa = 0, macs_fb = 0, macs_mv = 0, macs_vv = 0, macs_check = 0, macs_restart = 0;
  double flops_per_mac = 2.0;
  std::string to_json() const;
};

struct EigsOptions {
  int nev = 10;
  int m = 0;
  double tol = 1e-10;
  uint64_t seed = 0;
  int max_restarts = 100;
  int guard = 1;
  int max_guard = 64;
  double est_factor = 1e3;  // candidates are checked explicitly once est <= est_factor * tol
  int want_vectors = 0;
  int profile = 0;
};

struct EigsResult {
  bool converged = false;
  int nconv = 0, cycles = 0, guard_passes = 0;
  std::vector<std::complex<double>> lambda;
  std::vector<double> resid;
  std::vector<double> vec_re, vec_im;  // n x nev column-major
  int64_t launches = 0;
  double t_total_ms = 0, t_solve_ms = 0, t_orth_ms = 0;
  double max_restart_defect = 0;  // max ||H Q - Q T|| / ||H|| over restarts
  int64_t graph_launches = 0;     // one CUDA graph replay per Krylov-Schur cycle
  double t_ritz_ms = 0, t_check_ms = 0, t_restart_ms = 0, t_sync_ms = 0;  // host phase timers
};

// norms1 = {||K||_1, ||C||_1, ||M||_1} of the (scaled) pencil used by the
// operator.
EigsResult solve_quadratic_device(OperatorEngine& op, const EigsOptions& o, Ledger& L,
                                  const double norms1[3]);

}  // namespace rqb
