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
//
// Charges follow the reference operations one for one (the
// oracle's rq::spmv / dot / axpy call sequence): the GPU fuses and skips work
// (B-images kept beside the basis, one fused C/M SpMV) but the ledger counts
// the algorithm's operations, so its counters equal the reference CPU path's
// for the same operation (tests/test_gpu_parity.py ledger tests):
//   lu_factorize / build_operator  fa 1, sum over pivots of (nf-k-1)^2
//   apply_operator                 fb 1 (sum np^2 + 2 np (nf-np)), mv 3 (nnz), vv 3 (n)
//   B-product (b_inner, CGS)       mv 1 (nnz); each 2n dot or axpy: vv 1 (2n)
//   explicit residual check        check 1 per candidate (3 nnz)
//   restart V <- V Q               restart 1 (m p 2n)
struct Ledger {
  int64_t n_fa = 0, n_fb = 0, n_mv = 0, n_vv = 0, n_check = 0, n_restart = 0;
  double macs_fa = 0, macs_fb = 0, macs_mv = 0, macs_vv = 0, macs_check = 0, macs_restart = 0;
  double flops_per_mac = 2.0;
  std::string to_json() const;
  // counters as {ops, macs} x {fa, fb, mv, vv, check, restart}
  void get(double* out12) const;
  void add(const Ledger& o, bool with_fa);
};

// per-operation charges (see above) for the operator `op`
void charge_factor(Ledger& L, const OperatorEngine& op);
void charge_apply(Ledger& L, const OperatorEngine& op);
void charge_bproduct(Ledger& L, const OperatorEngine& op);  // one M-product (B = diag(I, M))
void charge_vv2n(Ledger& L, const OperatorEngine& op, int64_t count);  // count 2n-length dots / axpys

struct EigsOptions {
  int nev = 10;
  int m = 0;
  double tol = 1e-10;
  uint64_t seed = 0;
  int max_restarts = 100;
  int guard = 1;
  int max_guard = 64;
  int guard_single_cluster = 1;  // 0: run the guard pass even when every pair is one converged cluster
  double est_factor = 1e3;  // candidates are checked explicitly once est <= est_factor * tol
  int want_vectors = 0;
  int profile = 0;
  int block = 1;  // block Krylov-Schur block size (1: single-vector; 2..8: SURVEY.md §8 f2)
  int refine = 1;  // quadratic Rayleigh-quotient refinement of the returned eigenvalues
  int block_min_steps = 1;  // block mode: cycles with room for fewer block steps take width-1 steps (1: never)
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
