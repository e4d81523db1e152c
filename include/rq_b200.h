/* SPDX-License-Identifier: Apache-2.0
 *
 * rq_b200.h — C-ABI of the B200-native shift-invert quadratic eigensolver
 * (factor / solve / eigensolve path of arXiv 2112.14064, "Performance of rIGA
 * in solving quadratic eigenvalue problems").
 *
 * This is the drop-in boundary. The reference declares no factor/solve/eig
 * entry points in proj/include; they exist only as SPEC
 * operations. Each function below names the SPEC operation (or the reference
 * declaration) it replaces. The C++ wrappers in include/rigaqep/sparsela.hpp and
 * include/rigaqep/eig.hpp give those operations their SPEC signatures over the
 * reference's rq:: types and call this ABI.
 *
 * Conventions:
 *   - every function returns an int equal to an rq::errc value
 *     (reference proj/include/rigaqep/types.hpp:14-23); 0 = ok;
 *   - rq_last_error() returns the thread-local message of the last failure;
 *   - all array arguments are HOST pointers owned by the caller, copied in/out;
 *   - handles own their device memory and one CUDA stream; *_destroy frees it;
 *   - no exceptions cross the ABI; there is no CPU fallback: without a usable
 *     sm_100a device the numeric entry points fail with RQ_E_CONFIG.
 *   - FP64 real arithmetic: the GPU path accepts real pencils and real shifts
 *     only; complex input is rejected with RQ_E_CONFIG.
 */
#ifndef RQ_B200_H
#define RQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* rq::errc (types.hpp:14-23) */
enum {
  RQ_OK = 0,
  RQ_E_GENERIC = 1,
  RQ_E_CONFIG = 2,
  RQ_E_ASSEMBLY = 3,
  RQ_E_SOLVER = 4,
  RQ_E_VERIFICATION = 5,
  RQ_E_DOMAIN = 6,
  RQ_E_DIMENSION = 7,
  RQ_E_SINGULAR = 8
};

const char* rq_last_error(void);
const char* rq_version(void);
/* Select the CUDA device used by handles created afterwards on this thread
 * (one process per GPU: rank r calls rq_set_device(local_rank)). */
int rq_set_device(int device);

/* ------------------------------------------------------------------------ */
/* Input construction (host): spaces + BASELINE assembly.                   */
/* Replaces build_iga_space / build_riga_space / boundary_mask              */
/* (spaces.hpp:68-80) + SPEC assembly with the BASELINE   */
/* forms K = int(div.div | curl.curl) + phi.phi, M = int phi.phi,           */
/* C = alpha M + beta K, (p+1)^2 Gauss points, constrained DOFs eliminated. */
/* ------------------------------------------------------------------------ */
typedef struct rq_pencil rq_pencil_t;

enum { RQ_SPACE_CURL = 0, RQ_SPACE_DIV = 1 }; /* rq::SpaceKind (spaces.hpp:30) */

typedef struct {
  int kind;     /* RQ_SPACE_CURL or RQ_SPACE_DIV */
  int degree;   /* p >= 2 */
  int elems;    /* ne per direction (unit square) */
  int levels;   /* rIGA bisection levels L (0 = maximum-continuity IGA) */
  double alpha; /* Rayleigh damping C = alpha*M + beta*K */
  double beta;
} rq_space_desc;

int rq_pencil_assemble(const rq_space_desc* desc, rq_pencil_t** out);
/* The paper's vibroacoustic pencil (assemble_acoustic, SPEC.md:225-232;
 * PAPER.md:165-200, Fig. 8 material rho = 1, c = 340, alpha = 5e4, beta =
 * 200): H(div) space of `degree` on the unit square (rIGA levels as above),
 * u.n = 0 on the rigid edges, absorbing edges (bit mask: left 1, right 2,
 * bottom 4, top 8) free; K = int rho c^2 div u div v + int_GA alpha (u.n)(v.n),
 * C = int_GA beta (u.n)(v.n), M = int rho u.v; all real. Host assembly. */
int rq_pencil_assemble_acoustic(int degree, int elems, int levels, double rho, double c, double alpha, double beta,
                                int absorbing_edges, rq_pencil_t** out);
/* The paper's conductive electromagnetic pencil (assemble_em, SPEC.md:216-224;
 * PAPER.md §2.1): H(curl) space of `degree` on the unit square, E x n = 0; K =
 * int curl u (-1/mu) curl v, M = int eps u.v, C = -i D with D = int u . diag(
 * sigma_x(y), sigma_y(y)) v over nlayers horizontal layers (layers: nlayers x
 * {y0, y1, sigma_x, sigma_y}). The handle's C slot holds D (real); D_out (nnz,
 * nullable) receives a copy. Solve with rq_zeig_* (C = -i D is complex). */
int rq_pencil_assemble_em(int degree, int elems, int levels, double mu, double eps, int nlayers, const double* layers,
                          double* D_out, rq_pencil_t** out);
/* The same pencil, bit for bit, assembled on the current CUDA device
 * (pattern, per-element Gauss quadrature, colour-ordered
 * gather; no atomics). resident = 1 keeps K, C, M in device memory only
 * (rq_pencil_csr copies them out on demand; rq_operator_create_pencil uses
 * them in place); the pattern is always copied to the host. ms (nullable,
 * double[5]) receives the device ms of the three stages {pattern, element
 * matrices, gather}, then the host ms of the O(n) preparation (free
 * numbering, supports, Gauss tables) and of the copy back. */
int rq_pencil_assemble_device(const rq_space_desc* desc, int resident, rq_pencil_t** out, double* ms);
/* n_full = all DOFs, n_free = after BC elimination, nnz = shared-pattern nnz */
int rq_pencil_dims(const rq_pencil_t* p, int64_t* n_full, int64_t* n_free, int64_t* nnz);
/* Shared CSR pattern (rowptr int64[n+1], col int32[nnz], sorted per row) and
 * the three value arrays; any output pointer may be NULL. */
int rq_pencil_csr(const rq_pencil_t* p, int64_t* rowptr, int32_t* col, double* K, double* C,
                  double* M);
/* Per free DOF: inclusive element support box {x0, x1, y0, y1} (int32[4*n])
 * and the full-space DOF id (int64[n]); either may be NULL. */
int rq_pencil_supports(const rq_pencil_t* p, int32_t* box, int64_t* free_to_full);
void rq_pencil_destroy(rq_pencil_t* p);

/* Univariate / vector space bookkeeping exposed for parity with the
 * reference spaces code (spaces.cpp:33-113). */
int rq_space_dims(const rq_space_desc* desc, int64_t* nx_x, int64_t* ny_x, int64_t* nx_y,
                  int64_t* ny_y);
/* Sorted constrained full-space DOF ids (boundary_mask, spaces.cpp:79-113).
 * *count receives the number; mask may be NULL to query it. */
int rq_space_boundary_mask(const rq_space_desc* desc, int64_t* mask, int64_t* count);

/* ------------------------------------------------------------------------ */
/* Symbolic analysis (host C++): nested_dissection_order  */
/* + multifrontal front structure.                                          */
/* ------------------------------------------------------------------------ */
typedef struct rq_symbolic rq_symbolic_t;

typedef struct {
  int64_t n;
  int64_t nfronts;
  int64_t nlevels;       /* height-ordered batches (leaves = level 0) */
  int64_t max_front;     /* max nf */
  int64_t max_npiv;
  int64_t nnz_l;         /* stored lower-factor entries incl. diagonal */
  int64_t nnz_u;         /* stored upper-factor entries incl. diagonal */
  int64_t pool_doubles;  /* dense front pool size */
  double flops_lu;       /* F_LU = sum_f sum_k (nf-k-1) + 2 (nf-k-1)^2 (real) */
  double flops_schur;    /* sum_f 2 npiv (nf-npiv)^2 */
  double flops_schur_large; /* the same over fronts with nf >= 1024 */
  double trisolve_bytes; /* algorithmic bytes of one forward+backward solve */
} rq_symbolic_stats;

/* Geometric nested dissection over the DOF support boxes.
 * box: int32[4*n] as returned by rq_pencil_supports; elems: ne; leaf: max
 * DOFs in a leaf (default 64). */
int rq_nd_order(int64_t n, const int32_t* box, int elems, int leaf, rq_symbolic_t** out);
int rq_symbolic_stats_get(const rq_symbolic_t* s, rq_symbolic_stats* out);
/* perm[new] = old (free-DOF ids) */
int rq_symbolic_perm(const rq_symbolic_t* s, int32_t* perm);
/* Per front (postorder): parent (-1 root), npiv, nf, first pivot (new index),
 * level (height batch). Any array may be NULL. */
int rq_symbolic_fronts(const rq_symbolic_t* s, int32_t* parent, int32_t* npiv, int32_t* nf,
                       int32_t* start, int32_t* level);
/* Row list of front f (new indices, ascending; pivots first). */
int rq_symbolic_front_rows(const rq_symbolic_t* s, int64_t f, int32_t* rows);
void rq_symbolic_destroy(rq_symbolic_t* s);

/* ------------------------------------------------------------------------ */
/* Numeric multifrontal LU on the GPU: lu_factorize and   */
/* solve_factored.                                        */
/* ------------------------------------------------------------------------ */
typedef struct rq_factor rq_factor_t;

typedef struct {
  int64_t swaps;         /* off-diagonal pivots taken (threshold 0.1) */
  double factor_ms;      /* device time of the numeric factorization */
  double gflops;         /* flops_lu / factor time */
  int64_t launches;      /* kernels launched by one factorization */
} rq_factor_info;

/* A = Q(sigma) values on the shared pattern (free-DOF ordering). */
int rq_factor_create(const rq_symbolic_t* s, int64_t n, const int64_t* rowptr,
                     const int32_t* col, const double* aval, rq_factor_t** out);
/* Re-run the numeric factorization with new values on the same pattern (host
 * array of nnz doubles, CSR order; pinned memory lets the upload overlap the
 * factorization: the values stream up in chunks while the kernel runs). */
int rq_factor_refactor(rq_factor_t* f, const double* aval);
int rq_factor_get_info(const rq_factor_t* f, rq_factor_info* out);
/* x = A^{-1} b for nrhs right-hand sides (column-major n x nrhs, host).
 * Several right-hand sides go through the multi-RHS sweeps (up to 8 vectors
 * per pass over L and U). */
int rq_factor_solve(rq_factor_t* f, const double* b, double* x, int nrhs);
/* Same with an explicit sweep width: block = right-hand sides per pass over
 * the factors (1: the single-vector sweeps, 2..8: multi-RHS sweeps). */
int rq_factor_solve_ex(rq_factor_t* f, const double* b, double* x, int nrhs, int block);
/* Complex A = Are + i Aim on the pattern (rowptr, col) (Q(s)
 * over complex scalars, e.g. a complex shift): factored on the
 * GPU as its real-equivalent 2n system (unknowns 2k = Re x_k, 2k+1 = Im x_k,
 * i.e. the cdouble layout; 2 x 2 blocks [[Re a, -Im a], [Im a, Re a]]) by the
 * same multifrontal LU with threshold pivoting over the 2n unknowns. s2 is the
 * ordering of the 2n unknowns (rq_nd_order over the support boxes repeated
 * per unknown pair). Aim may be NULL (real). */
int rq_factor_create_complex(const rq_symbolic_t* s2, int64_t n, const int64_t* rowptr, const int32_t* col,
                             const double* are, const double* aim, rq_factor_t** out);
int rq_factor_refactor_complex(rq_factor_t* f, const double* are, const double* aim, const int64_t* rowptr,
                               const int32_t* col);
/* x = A^{-1} b for a complex factorization; b, x: nrhs interleaved {re, im}
 * vectors of n (cdouble[n] each). RQ_E_CONFIG on a real factorization. */
int rq_factor_solve_complex(rq_factor_t* f, const double* b, double* x, int nrhs);
/* Copy front f back: dense ld*nf column-major block holding L\U and the
 * Schur complement, ld = *ld_out; ipiv[npiv] local swap sequence. */
int rq_factor_front_export(const rq_factor_t* f, int64_t front, double* dense, int32_t* ipiv,
                           int64_t* ld_out);
/* Profiling run (not for timed steps): one un-graphed factorization with CUDA
 * events around every launch. Per kernel class {0 scatter, 1 extend_add,
 * 2 front_lu_smem, 3 panel_lu, 4 panel_apply, 5 schur_dmma}: device ms,
 * launches, algorithmic work (real flops; bytes for classes 0-1). */
int rq_factor_profile(rq_factor_t* f, double* ms, int64_t* launches, double* work);
/* Task-level profile of the persistent task-DAG factorization (profiling run):
 * out[3t+0] busy ms (summed over CTAs), out[3t+1] reserved (0), out[3t+2] task
 * count, for t = {SMALL, ASM, DIAG, ROWS, COLS, UPD (per-step updates)};
 * out[18] persistent grid size, out[19] tasks, out[20] ready-queue wait ms
 * summed over CTAs, out[21] UPDCB busy ms, out[23] UPDCB count. double[24]. */
int rq_factor_dag_profile(rq_factor_t* f, double* out);
/* Evidence entry (development): the contribution-block Schur update of ONE
 * front (front < 0: the largest), i.e. the factorization's own UPDCB task code
 * (C -= L21 U12 with K = npiv on FP64 tensor cores) as a plain grid, timed over
 * `reps` launches. Overwrites that front's contribution block: refactor after.
 * out[0] ms per launch, out[1] flops per launch, out[2] front, out[3] tiles,
 * out[4] K, out[5] grid. double[6]. */
int rq_factor_bench_updcb(rq_factor_t* f, int front, int reps, double* out);
void rq_factor_destroy(rq_factor_t* f);

/* ------------------------------------------------------------------------ */
/* Shift-invert operator of the linearised pencil: build_operator,          */
/* apply_operator, b_inner, arnoldi_run, solve_quadratic. */
/* Vectors of length 2n are (upper; lower) blocks, free-DOF ordering.       */
/* ------------------------------------------------------------------------ */
typedef struct rq_operator rq_operator_t;

typedef struct {
  double sigma;       /* real shift */
  int scaling;        /* 1: scale_pencil with varsigma = sqrt(maxabs K / maxabs M) */
} rq_operator_opts;

int rq_operator_create(int64_t n, const int64_t* rowptr, const int32_t* col, const double* K,
                       const double* C, const double* M, const rq_symbolic_t* s,
                       const rq_operator_opts* opts, rq_operator_t** out);
/* The same operator from a pencil handle: a device-resident pencil
 * (rq_pencil_assemble_device, resident = 1) is used in place — scaling,
 * Q(s) and the residual norms are formed on the device with the host path's
 * rounding, so the results equal rq_operator_create's on the same pencil. */
int rq_operator_create_pencil(const rq_pencil_t* p, const rq_symbolic_t* s,
                              const rq_operator_opts* opts, rq_operator_t** out);
double rq_operator_varsigma(const rq_operator_t* op);
/* r = L(s)^{-1} B v : r_u = -Q(s)^{-1}(s M v_u + C v_u + M v_l), r_l = s r_u + v_u
 * (of the possibly scaled pencil). */
int rq_operator_apply(rq_operator_t* op, const double* v, double* r);
/* x_u^T y_u + x_l^T M y_l */
int rq_operator_b_inner(rq_operator_t* op, const double* x, const double* y, double* out);
/* y = A x for A in {0: K, 1: C, 2: M, 3: Q(s)} (scaled pencil) */
int rq_operator_spmv(rq_operator_t* op, int which, const double* x, double* y);
/* m-step B-orthogonal Arnoldi with CGS2 from v1 (B-normalised inside).
 * V: (m+1) x 2n row-major, H: (m+1) x m column-major. */
int rq_operator_arnoldi(rq_operator_t* op, const double* v1, int m, double* V, double* H);
rq_factor_t* rq_operator_factor(rq_operator_t* op); /* borrowed */
/* Device time per call (CUDA events, device-resident buffers, after warm-up):
 * what = 0 apply_operator, 1 solve_factored, 2 fused C/M SpMV, 3 CGS GEMV-T
 * over `param` basis vectors, 4 GEMV-N over `param` vectors, 5 numeric
 * factorization (graph replay), 6 M SpMV, 7 restart DGEMM (2n x param) x
 * (param x param), 8 batched pencil residual of `param` candidates,
 * 9 block apply_operator of `param` (<= 8) vectors, 10 multi-RHS solve of
 * `param` (<= 8) right-hand sides.
 * what | 0x100: scrub L2 (256 MiB) before every call. */
int rq_operator_time(rq_operator_t* op, int what, int iters, int param, double* ms_per_call);
void rq_operator_destroy(rq_operator_t* op);

typedef struct {
  int nev;
  int m;              /* Krylov dimension; <= 0 selects 2*nev+1 (BASELINE) */
  double tol;         /* explicit pencil-residual tolerance */
  uint64_t seed;      /* splitmix64 start vector, uniform[-1,1] */
  int max_restarts;   /* default 100 */
  int guard;          /* completeness guard (deflated fresh restarts), 1 = on */
  int profile;        /* 1: time operator / orthogonalisation per step (synchronising) */
  int block;          /* block Krylov-Schur block size b (2..8; multi-RHS sweeps, block CGS2);
                         <= 1: single-vector Krylov-Schur */
} rq_eigs_opts;

typedef struct {
  int nconv;
  int restarts;       /* Krylov-Schur cycles (all passes) */
  int guard_passes;
  int64_t n_fa, n_fb, n_mv, n_vv, n_check, n_restart; /* ledger op counts */
  double macs_fa, macs_fb, macs_mv, macs_vv, macs_check, macs_restart;
  double t_total_ms, t_factor_ms, t_solve_ms, t_spmv_ms, t_orth_ms, t_host_ms;
  int64_t launches;
  double restart_defect; /* max ||H Q - Q T|| / ||H|| over restarts (exactness check) */
  double t_ritz_ms;      /* host: Schur form + Ritz vectors of H_m */
  double t_check_ms;     /* explicit pencil residuals (device + sync) */
  double t_restart_ms;   /* host restart basis + device V Q */
  double t_sync_ms;      /* host blocked on the Arnoldi-step graphs (device time) */
} rq_eigs_info;

/* solve_quadratic: nev eigenpairs of K + lam C + lam^2 M nearest sigma.
 * lam_re/lam_im/resid: double[nev]; vec_re/vec_im: n x nev column-major
 * (may be NULL). Returns RQ_E_SOLVER with the converged prefix filled when
 * max_restarts is exhausted. */
int rq_eigs_run(rq_operator_t* op, const rq_eigs_opts* opts, double* lam_re, double* lam_im,
                double* resid, double* vec_re, double* vec_im, rq_eigs_info* info);
/* The Krylov workspace (basis, B-images, pinned staging and the captured cycle
 * graphs: ~6 (m+1) 2n doubles, 9 GB at cfg4 with m = 201) stays with the
 * operator so repeated solves allocate nothing; this frees it (the next
 * rq_eigs_run rebuilds it). */
int rq_operator_release_workspace(rq_operator_t* op);
/* CostLedger::to_json-compatible snapshot (sparse.cpp:80-97) of the last run. */
int rq_eigs_ledger_json(const rq_operator_t* op, char* buf, size_t len);
/* The operator's cumulative CostLedger (reference sparse.hpp:57-103): every
 * operation since creation (build_operator's factorization: fa 1) or the last
 * reset. Charges follow the reference operations one for one:
 * apply_operator fb 1 + mv 3 + vv 3; b_inner mv 1 + vv 1; spmv mv 1; an Arnoldi
 * step apply + 3 B-products + (4(j+1)+1) 2n-vector dots/axpys; a residual check
 * per candidate; a restart per V Q. out: double[12] = {ops, macs} x {fa, fb,
 * mv, vv, residual_check, restart}. */
int rq_operator_ledger(const rq_operator_t* op, double* out);
int rq_operator_ledger_json(const rq_operator_t* op, char* buf, size_t len);
int rq_operator_ledger_reset(rq_operator_t* op);

/* scale_pencil: varsigma = sqrt(maxabs K /
 * maxabs M); the scaled pencil is (K, varsigma C, varsigma^2 M) with
 * eigenvalues gamma = lambda / varsigma. Cs, Ms (nnz, nullable) receive the
 * scaled values. Zero M -> RQ_E_DOMAIN. Host only. */
int rq_scale_pencil(int64_t nnz, const double* K, const double* C, const double* M, double* varsigma,
                    double* Cs, double* Ms);
/* ritz_extract: H (m+1) x m column-major (real, from
 * rq_operator_arnoldi or a restart), shift sigma and scaling varsigma of the
 * operator. For the m Ritz pairs in wanted order (nearest the shift first,
 * conjugate pairs adjacent, +imag first): theta (double[2m], re/im), lambda =
 * sigma + varsigma / theta (double[2m]), residual estimate |beta e_m^H y|
 * (double[m]) and y (m x m complex column-major, interleaved re/im: double[2m^2],
 * unit 2-norm). Any output may be NULL. QR non-convergence -> RQ_E_SOLVER.
 * Host only. */
int rq_ritz_extract(const double* H, int m, double sigma, double varsigma, double* theta, double* lam, double* est,
                    double* Y);
/* krylov_schur_restart: from an m-step decomposition
 * S V_m = V_m H_m + beta v_{m+1} e_m^T (V: (m+1) x 2n row-major host, H: (m+1) x m
 * column-major host), keep the `keep` wanted Ritz directions (closed under
 * conjugation; real orthonormal basis of their Schur vectors). On return
 * V[0..p] = {V_m Q_p, v_{m+1}} (V_m Q_p on the device, DMMA) and H holds
 * [T_p; b_p^T] in its leading (p+1) x p block, so S V_p = V_p T_p +
 * v_{p+1} b_p^T. keep >= m: identity restart (p = m). *p_out = p. */
int rq_operator_krylov_schur_restart(rq_operator_t* op, int m, int keep, double* V, double* H, int* p_out);

/* ------------------------------------------------------------------------ */
/* solve_generalized_hermitian (Alg. 1, Remark 3):  */
/* A u = lambda B u, A symmetric, B symmetric positive definite, one CSR      */
/* pattern, real shift s (the non-conductive Maxwell problem, Remark 2).      */
/* Shift-invert Lanczos with thick restarts on S = (A - s B)^{-1} B: A - s B  */
/* factored on the GPU (same multifrontal LU), N-vectors on the device,       */
/* symmetric tridiagonal (arrowhead after a restart) projected matrix, real   */
/* Ritz values, lambda = s + 1/theta. Converged on the explicit residual      */
/* ||A u - lambda B u|| / ((||A||_1 + |lambda| ||B||_1) ||u||) <= tol.        */
/* ------------------------------------------------------------------------ */
typedef struct rq_gh rq_gh_t;
typedef struct {
  int nev;
  int m;              /* Krylov dimension; <= 0: max(2 nev, nev + 20) */
  double tol;
  uint64_t seed;      /* splitmix64 start vector, uniform[-1,1] */
  int max_restarts;   /* <= 0: 100 */
} rq_gh_opts;
typedef struct {
  int nconv;
  int cycles;
  int restarts;
  double lanczos_defect; /* max |v_i^T B S v_j| over i < j-1 (three-term structure) / ||T|| */
  double sym_defect;     /* max |v_{j-1}^T B S v_j - beta_{j-1}| / ||T|| (symmetry of T) */
  int64_t launches;
  double t_total_ms;
} rq_gh_info;
int rq_gh_create(int64_t n, const int64_t* rowptr, const int32_t* col, const double* A, const double* B,
                 const rq_symbolic_t* s, double shift, rq_gh_t** out);
/* lam, resid: double[nev] (nearest the shift first); vec: n x nev column-major,
 * unit 2-norm (may be NULL). Non-convergence -> RQ_E_SOLVER. */
int rq_gh_run(rq_gh_t* h, const rq_gh_opts* opts, double* lam, double* resid, double* vec, rq_gh_info* info);
void rq_gh_destroy(rq_gh_t* h);

/* ------------------------------------------------------------------------ */
/* Complex pencils / complex shifts (SPEC.md:408-470 over complex scalars;  */
/* SURVEY.md §8 f4; the conductive EM pencil has C = -i sigma M_sigma):     */
/* K, C, M complex on one pattern (interleaved {re, im} per entry), complex */
/* shift s. Q(s) is factored on the GPU as its real-equivalent 2n system    */
/* (s2: ordering of the 2n unknowns, rq_nd_order over the boxes repeated    */
/* per (Re, Im) pair); complex Krylov-Schur with conjugated CGS2            */
/* projections on the device, complex Schur form of H_m on the host.        */
/* ------------------------------------------------------------------------ */
typedef struct rq_zeig rq_zeig_t;
int rq_zeig_create(const rq_symbolic_t* s2, int64_t n, const int64_t* rowptr, const int32_t* col, const double* K_c,
                   const double* C_c, const double* M_c, double s_re, double s_im, rq_zeig_t** out);
/* nev pairs nearest s: lam_c (interleaved, double[2 nev]), resid (double[nev]:
 * ||Q(lam) u|| / ((||K||_1 + |lam| ||C||_1 + |lam|^2 ||M||_1) ||u||)), vec_c (n x
 * nev complex, interleaved, may be NULL), stats {cycles, nconv}. Non-convergence
 * -> RQ_E_SOLVER. */
int rq_zeig_run(rq_zeig_t* h, int nev, int m, double tol, uint64_t seed, int max_restarts, double* lam_c,
                double* resid, double* vec_c, int32_t* stats);
void rq_zeig_destroy(rq_zeig_t* h);

/* ------------------------------------------------------------------------ */
/* Wire formats (reference sparse.cpp:121-174,         */
/* SPEC.md:269, 371, 503). Host only.                                       */
/* ------------------------------------------------------------------------ */
/* write_matrix_market: coordinate real|complex general, 1-based, "%.17g";  */
/* im may be NULL (real). Same bytes as the reference writer.               */
int rq_mm_write(int64_t n, const int64_t* rowptr, const int32_t* col, const double* re, const double* im,
                const char* path);
/* write_matrix_market_vector: array complex general, one "re im" per line  */
int rq_mm_write_vector(int64_t n, const double* re, const double* im, const char* path);
/* read_matrix_market: sorted CSR with duplicate entries summed
 * (from_triplets). Returns a handle; rq_mm_dims / rq_mm_csr copy it out.  */
typedef struct rq_mm rq_mm_t;
int rq_mm_read(const char* path, rq_mm_t** out);
int rq_mm_dims(const rq_mm_t* m, int64_t* n, int64_t* nnz, int* complex_values);
int rq_mm_csr(const rq_mm_t* m, int64_t* rowptr, int32_t* col, double* re, double* im);
void rq_mm_destroy(rq_mm_t* m);
/* Pencil export: <prefix>K.mtx, <prefix>C.mtx, <prefix>M.mtx */
int rq_pencil_write_mm(const rq_pencil_t* p, const char* prefix);
/* Eigenpair dump: JSON array of {re, im, residual}. *len
 * receives the length (without NUL); buf may be NULL to query it. */
int rq_eigenpairs_json(int n, const double* re, const double* im, const double* residual, char* buf,
                       int64_t cap, int64_t* len);

#ifdef __cplusplus
}
#endif

#endif /* RQ_B200_H */
