// SPDX-License-Identifier: Apache-2.0
// Device engines of the B200 build: the multifrontal factor (lu_factorize /
// solve_factored) and the shift-invert operator with its
// Krylov kernels. Host code talks to them through this
// header only; all device memory lives inside.
#pragma once

#include <cuda_runtime_api.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "host/common.hpp"

namespace rqb {

// Device-side description of one front (kept in sync with device.cuh).
struct FrontDev {
  int64_t off;        // pool offset (doubles), column-major ld x nf
  int64_t rows_off;   // into rows[]
  int64_t cbvec_off;  // forward-solve contribution vector
  int64_t inv_off;    // extend-add maps: nchild arrays of nf int32 (child-local row or -1)
  int32_t nf, npiv, ld, start;
  int32_t nchild, child0, child1, scratch;  // scratch: slot of panel inverses (-1 none)
  int64_t rel_off;    // child -> parent map: parent-local row of each CB row (nf - npiv int32)
};

void cuda_check(cudaError_t e, const char* what);
// dst[0, bytes) = src (host) on stream s, returns when the copy has completed;
// a large pageable source is staged through pinned buffers by the host threads
// (host/upload.cpp)
void upload_host_sync(void* dst, const void* src, size_t bytes, cudaStream_t s);

// Host setup phase timer (RQB_SETUP_TRACE=1: one stderr line per phase).
struct SetupTrace {
  const char* who;
  bool on;
  double t0;
  explicit SetupTrace(const char* w);
  void mark(const char* phase);
};

struct DeviceBuffer {
  void* p = nullptr;
  size_t bytes = 0;
  DeviceBuffer() = default;
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer();
  void alloc(size_t nbytes);
  void upload(const void* src, size_t nbytes, cudaStream_t s);
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Launch plan of one height batch.
struct LevelPlan {
  std::vector<int32_t> small;     // fronts factored whole in shared memory
  std::vector<int32_t> big;       // fronts factored by the blocked panel path
  std::vector<int32_t> with_kids; // fronts receiving an extend-add
  std::vector<int32_t> all;
  int small_nf = 0;               // max nf over `small`
  int big_maxnf = 0, big_maxpanels = 0, big_cluster = 1, big_maxrows = 0;
  int ea_maxnf = 0;
  int solve_maxnf = 0;
  // device offsets into FactorEngine::d_lists
  int64_t off_small = 0, off_big = 0, off_kids = 0, off_all = 0;
  std::vector<std::vector<int32_t>> panel_fronts;  // per panel step: active big fronts
  std::vector<int64_t> off_panel;
};

// Per-launch CUDA-event timer (profiling runs only; not used in timed steps).
struct KernelTimer {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  std::vector<int> kinds;
  void begin(cudaStream_t s, int kind);
  void end(cudaStream_t s);
  void collect(double* ms, int64_t* count, int nkinds);
};

// factor kernel classes: scatter, extend_add, front_lu_smem, panel_lu, panel_apply
// (+ net_rowperm), schur_dmma, factor_dag (persistent task-DAG kernel)
constexpr int kFactorKinds = 7;

struct DagPlan;
struct DagPlanDeleter {
  void operator()(DagPlan* p) const;
};
struct MSolvePlan;  // multi-RHS sweeps (cuda/msolve.cu)
struct MSolvePlanDeleter {
  void operator()(MSolvePlan* p) const;
};

struct FactorEngine {
  // one stream and one set of solve buffers per engine: the C-ABI entry points
  // that enqueue on them hold this lock from the first enqueue to the last
  // synchronisation, so concurrent solves on one factorization
  // are safe (serialised)
  std::mutex mu;
  // factorization schedule: persistent task-DAG kernel (default) or the
  // level-synchronous multi-launch path (RQB_FACTOR=level, kept for A/B runs)
  bool use_dag = true;
  bool dag_lazy = false;  // the DAG tasks zero + assemble their own regions (no pool memset / scatter launch)
  std::unique_ptr<DagPlan, DagPlanDeleter> dag;
  int dag_ntasks = 0;
  bool dag_prof_enabled = false;
  Symbolic sym;
  int64_t n = 0, nnz = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaStream_t stream_up = nullptr;  // streamed upload of the values (factor_streamed)
  cudaEvent_t ev_up = nullptr;
  DeviceBuffer d_arrived;            // int: chunks of the upload sequence present in d_aval
  int* h_marks = nullptr;            // pinned: 1, 2, ... (the arrival counter's values)
  int n_marks = 0;
  int64_t stream_chunk = 1 << 21;    // values per chunk (16 MiB)
  std::vector<int32_t> chunk_order;  // upload sequence (rqb_dag_build: by the first task needing each chunk)
  DeviceBuffer d_pool, d_aval, d_qdst, d_rows, d_fronts, d_inv, d_ipiv, d_lists, d_scratch, d_rel;
  std::vector<int32_t> rel_h;  // concatenated child -> parent row maps
  DeviceBuffer d_flags;   // [0] singular, [1] swaps
  DeviceBuffer d_y, d_xnew, d_cbvec, d_perm;  // solve workspaces (n, n, cbvec), perm[new] = old
  // sync-free solve: work items, per-front item counts, dependency counters,
  // net row permutation of each front's pivot block
  DeviceBuffer d_items_fwd, d_items_bwd, d_rowperm, d_sf, d_ech, d_gsrc;
  // inverses of the pivot blocks' 64x64 diagonal tiles (computed after each
  // factorization): per block an nr x nr column-major square, strictly lower =
  // inv(L11) (unit diagonal implied), upper = inv(U11); d_dblk lists the blocks
  DeviceBuffer d_dinv, d_dblk, d_bpart;
  int n_dblk = 0;
  // dataflow state of the two sweeps in one int32 buffer (template + live
  // copy, reset by one D2D copy per solve): front deps fwd/bwd, ready queues
  // fwd/bwd, {head, tail} x2, per-front published/finished counters
  DeviceBuffer d_state0, d_state, d_sweep_stall;
  int64_t st_dep_fwd = 0, st_dep_bwd = 0, st_q_fwd = 0, st_q_bwd = 0, st_qctl = 0, st_cnt = 0;
  int n_fwd_items = 0, n_bwd_items = 0, solve_grid = 148, sweep_occ = 2, win_f = 8, win_b = 8;
  // multi-RHS sweeps: items, dataflow state and interleaved workspaces (built on first use)
  std::unique_ptr<MSolvePlan, MSolvePlanDeleter> mplan;
  std::vector<FrontDev> fronts_h;
  std::vector<LevelPlan> plans;
  int64_t nscratch = 0;
  double last_ms = 0.0;
  int64_t last_swaps = 0;
  int64_t launches_factor = 0, launches_solve = 0;
  cudaGraph_t graph_factor = nullptr;
  cudaGraphExec_t graph_factor_exec = nullptr;

  // rowptr/col: host pattern; rowptr_dev/col_dev: optional device copy of it
  // (the scatter map is built on the device); aval: host values or nullptr
  // (then set_values_device before factor()).
  FactorEngine(const Symbolic& s, int64_t n, const int64_t* rowptr, const int32_t* col,
               const double* aval, const int64_t* rowptr_dev = nullptr,
               const int32_t* col_dev = nullptr);
  ~FactorEngine();
  // Numeric factorization of the values currently in d_aval (device time in
  // last_ms). Returns the singular flag.
  void factor();
  void set_values(const double* aval_host);
  // set_values + factor with the upload overlapped: the values go up in CSR
  // order in chunks on a second stream while the task-DAG kernel runs; a task
  // waits until its own entries have arrived (lazy assembly only; otherwise
  // upload, then factor)
  void factor_streamed(const double* aval_host);
  void launch_factor_graph();
  void finish_factor();
  bool streaming = false;
  void set_values_device(const double* aval_dev);
  // x = A^{-1} b on device vectors (original ordering), enqueued on `stream`.
  void solve_device(const double* b, double* x, double scale_out = 1.0);
  // raise errc::solver if a triangular sweep hit its stall watchdog (syncs the stream)
  void check_sweeps();
  void enqueue_factor(KernelTimer* kt = nullptr);
  // One un-graphed factorization with per-launch events: device ms, launch
  // count and algorithmic work (flops; bytes for classes 0-1) per kernel class.
  void profile(double* ms, int64_t* count, double* flops);
};

// Enqueue forward+backward substitution on fe.stream: x = scale * A^{-1} b and,
// when xl != nullptr, xl = sigma * x + vu (fused lower block of apply_operator).
void rqb_solve_enqueue(FactorEngine& fe, const double* b, double* x, double scale,
                       const double* vu, double sigma, double* xl);
// Multi-RHS sweeps (up to 8 vectors, cuda/msolve.cu): for j < nrhs,
// x[:, j] = scale * A^{-1} b[:, j] (columns at ldb / ldx) and, when xl !=
// nullptr, xl[:, j] = sigma * x[:, j] + vu[:, j] (ldx / ldv). L and U are
// streamed once for all nrhs vectors.
// b[i * b_row_stride + j * ldb]: column-major right-hand sides (stride 1) or
// row-interleaved ones (b_row_stride = width, ldb = 1).
void rqb_msolve_enqueue(FactorEngine& fe, const double* b, int64_t ldb, int nrhs, double* x, int64_t ldx,
                        double scale, const double* vu, int64_t ldv, double sigma, double* xl,
                        int64_t b_row_stride = 1);
// build the multi-RHS sweep plan now (not during a stream capture)
void rqb_msolve_prepare(FactorEngine& fe);
// raise errc::solver if a multi-RHS sweep hit its stall watchdog (syncs the stream)
void rqb_msolve_check(FactorEngine& fe);
void rqb_solve_set_attrs(int maxnf);
void rqb_solve_prepare(FactorEngine& fe);
void rqb_dag_build(FactorEngine& fe);
void rqb_dag_enqueue(FactorEngine& fe);
void rqb_dag_profile(FactorEngine& fe, double* out);
void rqb_dag_bench_updcb(FactorEngine& fe, int front, int reps, double* out);
void rqb_rowperm_enqueue(FactorEngine& fe);
// X = V Q on FP64 tensor cores (csrc/cuda/gemm.cu): V n2 x k (vector j at
// V + j ldv), Q k x c column-major, X column-major (ldx >= n2) or row-major.
void vq_gemm(const double* V, int64_t ldv, int64_t n2, int k, const double* Q, int ldq, int c, double* X,
             int64_t ldx, bool row_major_out, cudaStream_t stream);
std::string rqb_dag_stall_report(FactorEngine& fe);

// Device-resident pencil (device assembly): CSR pattern and
// K, C, M values in HBM of the device that assembled them.
struct DevicePencil {
  int64_t n = 0, nnz = 0;
  int device = 0;
  DeviceBuffer d_rowptr, d_col, d_val;  // d_val: K | C | M, nnz each
  const double* K() const { return d_val.as<double>(); }
  const double* C() const { return d_val.as<double>() + nnz; }
  const double* M() const { return d_val.as<double>() + 2 * nnz; }
};

// Shift-invert operator on the linearised pencil, real FP64, device resident.
struct OperatorEngine {
  int64_t n = 0, nnz = 0;
  double sigma = 0.0, varsigma = 1.0;  // shift of the (scaled) pencil, scaling factor
  std::unique_ptr<FactorEngine> fac;
  DeviceBuffer d_rowptr, d_col, d_K, d_C, d_M, d_Q;
  DeviceBuffer d_w, d_t, d_part, d_scal;  // workspaces
  // Krylov-Schur workspace kept across solve_quadratic calls (eigs.cpp
  // EigWorkspace: basis buffers + the cycle graphs captured over them)
  std::shared_ptr<void> eig_ws;
  DeviceBuffer d_rcand, d_rpart;          // batched residual candidates / partials
  DeviceBuffer d_tb, d_bpart;             // block Krylov: SpMM output (n x 8), block-projection partials
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  int64_t nparts = 0;
  int64_t gemv_t_chunk = 256;  // CGS projection: entries per block, blocks
  int gemv_t_blocks = 1;

  // From host arrays (uploaded once; varsigma, C / M scaling, Q(s) and the
  // 1-norms, when norms1 is given, formed on the device as below).
  OperatorEngine(int64_t n, const int64_t* rowptr, const int32_t* col, const double* K,
                 const double* C, const double* M, const Symbolic& s, double sigma,
                 bool scaling, double* norms1 = nullptr);
  // From a device-resident pencil (host copy of the pattern for the symbolic
  // scatter maps): scaling, C/M scaling, Q(s) and the 1-norms of K, vC, v^2 M
  // (norms1) are formed on the device with the host constructor's rounding.
  OperatorEngine(const DevicePencil& dp, const int64_t* rowptr_h, const int32_t* col_h,
                 const Symbolic& s, double sigma, bool scaling, double* norms1);
  ~OperatorEngine();
  static std::unique_ptr<DevicePencil> upload_pencil(int64_t n, const int64_t* rowptr, const int32_t* col,
                                                     const double* K, const double* C, const double* M);
  // Device vector ops (2n vectors: upper; lower), all enqueued on `stream`.
  void spmv(int which, const double* x, double* y);          // y = A x
  void apply(const double* v, double* r);                    // r = L(s)^{-1} B v
  void bvec(const double* r, double* w);                     // w = [r_u; M r_l]
  // h[0..k) = V[0..k)^T w (V row-major k x 2n), deterministic two-stage reduction
  void gemv_t(const double* V, int k, const double* w, double* h);
  // r -= V[0..k)^T-combination: r -= sum_i h[i] V[i]; optionally h_acc += h
  void gemv_n(const double* V, int k, const double* h, double* r, double* h_acc);
  // out = ||r||_B computed with w = B r; v_next = r / out
  void bnorm_normalize(const double* r, const double* w, double* beta_out, double* v_next);
  // beta = ||r||_B with B r from one M-product; v_next = r / beta, bv_next = B r / beta
  void bnorm_normalize_b(const double* r, double* beta_out, double* v_next, double* bv_next);
  void dot2n(const double* x, const double* y, double* out);  // out = x.y (2n)
  // Block Krylov-Schur (bs <= 8 vectors, column j at V + j 2n):
  // R[:, j] = L(s)^{-1} B V[:, j] through the multi-RHS sweeps
  void apply_block(const double* V, int bs, double* R);
  // Wl[:, j] = M R_l[:, j] for the w block members (R: 2n columns at stride 2n; Wl: n x w, ld n)
  void mspmv_block(const double* R, int w, double* Wl);
  // r[e] -= sum_{i<k} V[i ldv + e] h[i] for e < len
  void gemv_n_len(const double* V, int k, int64_t ldv, int64_t len, const double* h, double* r);
  // beta = ||r||_B from the tracked wl = M r_l; v_next = r / beta, bv_next = [r_u; wl] / beta
  void bnorm_normalize_w(const double* r, const double* wl, double* beta_out, double* v_next, double* bv_next);
  // allocate what apply_block / gemm_t need for bases up to kmax vectors (outside graph captures)
  void prepare_block(int kmax, int bs);
  // H[i + j ldh] = V[:, i] . R[:, j] for i < k, j < bs (deterministic two-stage reduction)
  void gemm_t(const double* V, int k, const double* R, int bs, double* H, int ldh);
  // R[:, j] -= sum_{i<k} V[:, i] H[i + j ldh], j < bs
  void gemm_n(const double* V, int k, const double* H, int ldh, double* R, int bs);
  // Vout[c] = sum_k V[k] Q[k + c*ldq] for c < ncols (restart compression)
  void combine(const double* V, int k, const double* Q_dev, int ldq, int ncols, double* Vout);
  // Ritz vectors X = V^T-combination with Y (m x 2nc: columns Re y_c, Im y_c),
  // stored row-major in Xrm (2n x 2nc), and their pencil residuals:
  // out[2c] = ||Q(lambda_c) x_c||^2, out[2c+1] = ||x_c||^2 over block blk[c]
  // (lam: host {re, im} pairs of the scaled-pencil eigenvalues).
  // out[2nc + 6c ..] = u^H K u, u^H C u, u^H M u (re, im) of candidate c on its block (the
  // quadratic Rayleigh quotient's coefficients); out needs 8 nc doubles
  void ritz_residuals(const double* V, int m, const double* Y, int nc, const double* lam, const int* blk,
                      double* Xrm, double* out);
  // the same residuals (and coefficients) of the last batch in Xrm for new eigenvalues lam
  // (host {re, im} pairs; blocks as in the last ritz_residuals call)
  void residuals_again(const double* Xrm, int nc, const double* lam, double* out);
  // contiguous copy (n entries) of part (0 re, 1 im) of Ritz vector c of the
  // last ritz_residuals batch, block blk[c]
  void ritz_extract(const double* Xrm, int nc, int c, int part_im, double* out);
  // Average device ms of one call of an operation (see rq_operator_time).
  double time_op(int what, int iters, int param);

 private:
  void init_workspaces();
};

// Generalized Hermitian-definite problem A u = lambda B u (SPEC.md:471-479,
// solve_generalized_hermitian): A symmetric, B symmetric positive definite on
// one CSR pattern, real shift s. The device holds A, B and the factorization
// of A - s B; S = (A - s B)^{-1} B is B-self-adjoint, so its Krylov
// decomposition is a Lanczos one (host driver: host/lanczos.cpp).
struct GhEngine {
  int64_t n = 0, nnz = 0;
  double shift = 0.0;
  std::unique_ptr<FactorEngine> fac;
  DeviceBuffer d_rowptr, d_col, d_A, d_B, d_t, d_part, d_res;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  int64_t gemv_t_chunk = 256;
  int gemv_t_blocks = 1;
  GhEngine(int64_t n, const int64_t* rowptr, const int32_t* col, const double* A, const double* B,
           const Symbolic& s, double shift);
  void spmv(int which, const double* x, double* y);  // which 0: A, 1: B
  void apply(const double* v, double* r);            // r = (A - s B)^{-1} B v
  void gemv_t(const double* V, int k, const double* w, double* h);  // h = V[0..k)^T w
  void gemv_n(const double* V, int k, const double* h, double* r);  // r -= V[0..k) h
  // w = B r (one SpMV), beta = sqrt(r . w) -> *beta_out, v = r / beta, bv = w / beta
  void bnorm_normalize(const double* r, double* beta_out, double* v, double* bv);
  // out[2c] = ||A x_c - lam_c B x_c||^2, out[2c+1] = ||x_c||^2 for the nc
  // column-major vectors X (ld n)
  void residuals(const double* X, int nc, const double* lam_host, double* out_host);
};

}  // namespace rqb
