// SPDX-License-Identifier: Apache-2.0
// solve_quadratic (defaults :489-497; Alg. 2,
// :555-589): Krylov-Schur on the shift-invert operator of the linearised
// pencil with B-orthogonal CGS2 Arnoldi. The host owns the loop and the m x m
// projected problem; every N-sized vector lives on the device and stays real
// (real shift, real start vector).
//
// Per Arnoldi step:
//   r = S v_j                          (fused SpMV -> trisolve -> axpy)
//   2 x { w = B r; h = V^T w; r -= V h }   (CGS2)
//   beta = ||r||_B; v_{j+1} = r / beta
// Per cycle: complex Schur form of H_m, Ritz values theta, lambda = s + 1/theta
// (unscaled by varsigma), explicit pencil residuals of candidate pairs
// (SURVEY App. B D5), restart keeping keep = nev + min(20, m - nev - 1)
// wanted directions.
// Completeness guard: once nev pairs converge they are kept
// (deflated, b = 0) and the Krylov space is restarted from a fresh seeded vector
// B-orthogonalised against them; any newly converged Ritz value closer to the
// shift than the worst kept one is swapped in; repeat until a pass changes
// nothing.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <numeric>
#include <sstream>

#include "../engine.hpp"
#include "dense.hpp"
#include "eigs.hpp"

namespace rqb {

namespace {

struct Ritz {
  cplx theta;
  cplx lambda;  // unscaled
  double est;
  int idx;      // position in the (unreordered) Schur form
};

double dist(const cplx& l, double sigma) { return std::abs(l - sigma); }

constexpr double kClusterGap = 1e-4;  // relative Ritz-value gap below which values are one group

}  // namespace

std::string Ledger::to_json() const {
  std::ostringstream os;
  os.precision(17);
  auto cat = [&](const char* name, int64_t ops, double macs, bool last = false) {
    os << "  \"" << name << "\": {\"ops\": " << ops << ", \"macs\": " << macs
       << ", \"flops\": " << flops_per_mac * macs << "}" << (last ? "\n" : ",\n");
  };
  os << "{\n";
  cat("fa", n_fa, macs_fa);
  cat("fb", n_fb, macs_fb);
  cat("mv", n_mv, macs_mv);
  cat("vv", n_vv, macs_vv);
  cat("residual_check", n_check, macs_check);
  cat("restart", n_restart, macs_restart);
  os << "  \"flops_per_mac\": " << flops_per_mac << ",\n";
  os << "  \"total_flops\": " << flops_per_mac * (macs_fa + macs_fb + macs_mv + macs_vv) << "\n}";
  return os.str();
}

void Ledger::get(double* out) const {
  const int64_t ops[6] = {n_fa, n_fb, n_mv, n_vv, n_check, n_restart};
  const double macs[6] = {macs_fa, macs_fb, macs_mv, macs_vv, macs_check, macs_restart};
  for (int c = 0; c < 6; ++c) out[2 * c] = static_cast<double>(ops[c]), out[2 * c + 1] = macs[c];
}

void Ledger::add(const Ledger& o, bool with_fa) {
  if (with_fa) n_fa += o.n_fa, macs_fa += o.macs_fa;
  n_fb += o.n_fb, macs_fb += o.macs_fb;
  n_mv += o.n_mv, macs_mv += o.macs_mv;
  n_vv += o.n_vv, macs_vv += o.macs_vv;
  n_check += o.n_check, macs_check += o.macs_check;
  n_restart += o.n_restart, macs_restart += o.macs_restart;
}

void charge_factor(Ledger& L, const OperatorEngine& op) {
  double macs = 0;
  for (const Front& F : op.fac->sym.fronts)
    for (int k = 0; k < F.npiv; ++k) {
      const double r = F.nf - k - 1.0;
      macs += r * r;
    }
  L.n_fa += 1;
  L.macs_fa += macs;
}

void charge_apply(Ledger& L, const OperatorEngine& op) {
  double fb = 0;
  for (const Front& F : op.fac->sym.fronts) {
    const double np = F.npiv, nf = F.nf;
    fb += np * np + 2.0 * np * (nf - np);
  }
  L.n_fb += 1;
  L.macs_fb += fb;
  L.n_mv += 3;  // C v_u, M v_u, M v_l
  L.macs_mv += 3.0 * static_cast<double>(op.nnz);
  L.n_vv += 3;  // + s M v_u, + M v_l, r_l = s r_u + v_u
  L.macs_vv += 3.0 * static_cast<double>(op.n);
}

void charge_bproduct(Ledger& L, const OperatorEngine& op) {
  L.n_mv += 1;
  L.macs_mv += static_cast<double>(op.nnz);
}

void charge_vv2n(Ledger& L, const OperatorEngine& op, int64_t count) {
  L.n_vv += count;
  L.macs_vv += static_cast<double>(count) * 2.0 * static_cast<double>(op.n);
}

// pinned: the cycle's H / beta copies are truly asynchronous, so the host
// can start on them while the GPU already applies the operator to the
// continuation vector of the next cycle
struct Pinned {
  double* p = nullptr;
  explicit Pinned(size_t n) {
    cuda_check(cudaMallocHost(reinterpret_cast<void**>(&p), sizeof(double) * std::max<size_t>(n, 1)), "pinned");
  }
  Pinned(const Pinned&) = delete;
  Pinned& operator=(const Pinned&) = delete;
  ~Pinned() { cudaFreeHost(p); }
  double& operator[](size_t i) { return p[i]; }
  double* data() { return p; }
};

// Krylov-Schur workspace kept by the operator across solve_quadratic calls
// (OperatorEngine::eig_ws): the basis buffers and the cycle graphs captured
// over them stay valid as long as m does; no allocation, free or graph build
// in a repeated solve.
struct EigWorkspace {
  int m = -1, bs = 1;
  int64_t n2 = 0;
  DeviceBuffer dV, dV2, dBV, dBV2, dR, dW, dHa, dHb, dBeta, dQ, dX, dRes;
  DeviceBuffer dHc, dHd, dBeta2;  // block mode: second intra-block sub-passes, R2 diagonal
  DeviceBuffer dWl;               // block mode: tracked M r_l of the block members (n x bs)
  Pinned ha, hb, betas;
  Pinned hc, hd, betas2;
  Pinned hv, hq, hy;  // staging of the host -> device copies (start vectors, restart Q, Ritz Y)
  // cycle graph per (start index, basis buffer) and the kernels it launches
  std::map<std::pair<int, const double*>, std::pair<cudaGraphExec_t, int64_t>> graphs;
  // basis of m + bs vectors (m accounted by H, a frontier block of bs), H
  // (m + bs) x (m + bs) column-major
  EigWorkspace(int m_, int64_t n2_, int bs_)
      : m(m_), bs(bs_), n2(n2_), ha(static_cast<size_t>(m_ + bs_) * (m_ + bs_)),
        hb(static_cast<size_t>(m_ + bs_) * (m_ + bs_)), betas(m_ + bs_),
        hc(bs_ > 1 ? static_cast<size_t>(m_ + bs_) * (m_ + bs_) : 1),
        hd(bs_ > 1 ? static_cast<size_t>(m_ + bs_) * (m_ + bs_) : 1), betas2(m_ + bs_),
        hv(static_cast<size_t>(n2_)), hq(static_cast<size_t>(m_ + 1) * (2 * m_ + 2)),
        hy(static_cast<size_t>(m_ + 1) * (2 * m_ + 2)) {
    dV.alloc(sizeof(double) * (m + bs) * n2);
    dV2.alloc(sizeof(double) * (m + bs) * n2);
    dBV.alloc(sizeof(double) * (m + bs) * n2);
    dBV2.alloc(sizeof(double) * (m + bs) * n2);
    dR.alloc(sizeof(double) * n2 * bs);
    dW.alloc(sizeof(double) * n2);
    dHa.alloc(sizeof(double) * (m + bs) * (m + bs));
    dHb.alloc(sizeof(double) * (m + bs) * (m + bs));
    dBeta.alloc(sizeof(double) * (m + bs));
    if (bs > 1) {
      dHc.alloc(sizeof(double) * (m + bs) * (m + bs));
      dHd.alloc(sizeof(double) * (m + bs) * (m + bs));
      dBeta2.alloc(sizeof(double) * (m + bs));
      dWl.alloc(sizeof(double) * (n2_ / 2) * bs);
    }
    dQ.alloc(sizeof(double) * (m + 1) * (2 * m + 2));
    dX.alloc(sizeof(double) * n2 * 2 * (m + 1));
    dRes.alloc(sizeof(double) * 8 * (m + bs + 1));
  }
  ~EigWorkspace() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.first);
  }
};

EigsResult solve_quadratic_device(OperatorEngine& op, const EigsOptions& o, Ledger& L,
                                  const double norms1[3]) {
  using clock = std::chrono::steady_clock;
  const auto t0 = clock::now();
  const int64_t n = op.n, n2 = 2 * n;
  const int nev = o.nev;
  const int m = o.m > 0 ? o.m : 2 * nev + 1;
  if (nev < 1) fail(errc::config, "nev must be positive");
  if (m <= nev) fail(errc::config, "Krylov dimension m must exceed nev");
  if (m > 512) fail(errc::config, "Krylov dimension above 512");
  const int bs = std::max(1, o.block);  // block size (1: single-vector Krylov-Schur)
  if (bs > 8) fail(errc::config, "block size above 8");
  if (m + bs > n2) fail(errc::config, "Krylov dimension must be below 2N");
  if (m < nev + bs) fail(errc::config, "block Krylov-Schur needs m >= nev + block");
  if (!(o.tol > 0)) fail(errc::config, "tolerance must be positive");
  const int LDH = m + bs;  // leading dimension of H (rows: m accounted + the frontier block)
  // Step plan of a cycle from k accounted vectors (block mode): steps of width
  // bs while the cycle has room for at least block_min_steps of them, else
  // width 1 (the banded "sliding window" form of block Arnoldi: S applied to
  // the oldest frontier vector, projected against everything incl. the rest of
  // the frontier). Every step of width w applies S to V[j, j+w), projects
  // against V[0, j+bs) and appends V[j+bs, j+bs+w); the cycle always ends at
  // m accounted vectors with a frontier of bs.
  const int min_steps = std::getenv("RQB_BLOCK_MINSTEPS") ? std::max(1, std::atoi(std::getenv("RQB_BLOCK_MINSTEPS")))
                                                          : o.block_min_steps;
  auto plan_steps = [&](int k0) {
    std::vector<std::pair<int, int>> pl;
    const int w = (bs > 1 && (m - k0) >= bs * min_steps) ? bs : 1;
    for (int j = k0; j < m; j += w) pl.emplace_back(j, std::min(w, m - j));
    return pl;
  };
  const int keep_target = nev + std::min(20, m - nev - 1);
  const double sig = op.sigma;  // scaled shift
  const double vs = op.varsigma;
  cudaStream_t st = op.stream;

  EigsResult res;
  const int64_t launches0 = op.launches;
  // ledger: one factorization (already done when the operator was built)
  charge_factor(L, op);
  const double nnz = static_cast<double>(op.nnz);

  // V: Krylov basis; BV = B V kept alongside, so every B-inner product of CGS2
  // is a plain projection h = (BV)^T r (B = diag(I, M) symmetric) and each
  // step needs one M-product (for the new vector) instead of three
  EigWorkspace* wsp = static_cast<EigWorkspace*>(op.eig_ws.get());
  if (!wsp || wsp->m != m || wsp->n2 != n2 || wsp->bs != bs) {
    op.eig_ws.reset();
    auto fresh = std::make_shared<EigWorkspace>(m, n2, bs);
    wsp = fresh.get();
    op.eig_ws = fresh;
  }
  EigWorkspace& W = *wsp;
  if (bs > 1) op.prepare_block(m + bs, bs);  // sweep plan + block workspaces before any graph capture
  DeviceBuffer &dV = W.dV, &dV2 = W.dV2, &dBV = W.dBV, &dBV2 = W.dBV2, &dR = W.dR, &dW = W.dW, &dHa = W.dHa, &dHb = W.dHb,
               &dBeta = W.dBeta, &dQ = W.dQ, &dX = W.dX, &dRes = W.dRes, &dHc = W.dHc, &dHd = W.dHd,
               &dBeta2 = W.dBeta2;
  double* V = dV.as<double>();
  double* V2 = dV2.as<double>();
  double* BV = dBV.as<double>();
  double* BV2 = dBV2.as<double>();
  double* r = dR.as<double>();

  cudaEvent_t e_a, e_b;
  cuda_check(cudaEventCreate(&e_a), "event");
  cuda_check(cudaEventCreate(&e_b), "event");

  // Start block: vector i = splitmix64(seed + i * golden) uniform[-1,1]^{2N}
  // (i = 0: the single-vector start), B-orthogonalised (CGS2) against the
  // nlock vectors before it and the earlier members of the block, B-normalised
  // into V[nlock + i].
  auto fresh_block = [&](uint64_t seed, int nlock, int count) {
    for (int b = 0; b < count; ++b) {
      const int nb = nlock + b;
      std::vector<double> v(n2);
      uint64_t s = seed + 0x9E3779B97F4A7C15ull * static_cast<uint64_t>(b);
      for (int64_t i = 0; i < n2; ++i) v[i] = splitmix_uniform(s);
      cuda_check(cudaStreamSynchronize(st), "sync staging");  // the pinned staging buffer is free again
      std::memcpy(W.hv.data(), v.data(), sizeof(double) * n2);
      cuda_check(cudaMemcpyAsync(r, W.hv.data(), sizeof(double) * n2, cudaMemcpyHostToDevice, st), "H2D v0");
      for (int pass = 0; pass < 2 && nb > 0; ++pass) {
        op.gemv_t(BV, nb, r, dHa.as<double>());
        op.gemv_n(V, nb, dHa.as<double>(), r, nullptr);
        charge_bproduct(L, op);  // ledger: the reference algorithm's B-product
        charge_vv2n(L, op, 2 * nb);
      }
      op.bnorm_normalize_b(r, dBeta.as<double>() + LDH - 1, V + static_cast<int64_t>(nb) * n2,
                           BV + static_cast<int64_t>(nb) * n2);
      charge_bproduct(L, op);
      charge_vv2n(L, op, 1);
    }
  };

  std::vector<double> H(static_cast<size_t>(LDH) * m, 0.0);  // column-major (m+bs) x m
  auto Hc = [&](int i, int j) -> double& { return H[i + static_cast<size_t>(j) * LDH]; };

  fresh_block(o.seed, 0, bs);
  int k = 0;
  int cycles = 0, guard_passes = 0, pass_cycles = 0;
  bool converged_final = false;
  std::vector<double> prev_guard_dists;
  std::vector<Ritz> final_set, last_cand;
  std::vector<double> final_res, last_res;
  std::vector<int> final_block;  // 0 upper, 1 lower
  std::vector<double> final_vecs_re, final_vecs_im;
  Pinned &ha = W.ha, &hb = W.hb, &betas = W.betas;
  cudaEvent_t e_h;
  cuda_check(cudaEventCreateWithFlags(&e_h, cudaEventDisableTiming), "event");
  bool pre_applied = false;  // r already holds apply(V[k]) (speculative, see below)
  double t_solve = 0, t_orth = 0, t_ritz = 0, t_check = 0, t_restart = 0, t_sync = 0;
  double t_reorder = 0, t_basis = 0, t_host = 0;  // trace only: restart split, host time per cycle
  double check_gate = o.est_factor * o.tol;
  int last_nchk = 0;  // candidates of the last explicit check (row-major Ritz batch in dX)
  std::vector<double> last_lam, last_rq;  // that batch's scaled eigenvalues and Rayleigh-quotient coefficients
  int since_check = 0;
  int recheck_wait = 8;  // cycles before an ungated re-check (shorter when the last check was close)
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms_since = [](std::chrono::steady_clock::time_point a) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
  };
  double t_graph_build = 0;
  static const bool trace_cycles = std::getenv("RQB_EIGS_TRACE") != nullptr;  // per-cycle stderr line
  const double t_setup = ms_since(t0);
  auto& graphs = W.graphs;

  while (true) {
    // max_restarts bounds each Krylov-Schur pass (the main run and every guard
    // pass restart the count)
    if (pass_cycles >= o.max_restarts) break;
    ++cycles;
    ++pass_cycles;
    // ---- Arnoldi steps k .. m-1: one CUDA graph per (start, basis buffer) ----
    // block step at kc (bs = 1: an Arnoldi step): R = S V[kc, kc+bs); CGS2
    // against V[0, kt), kt = kc + bs (block projections: every basis vector
    // read once per pass for the whole block); then the block's own
    // Gram-Schmidt (CGS2 against its earlier members) and B-normalisation into
    // V[kt + j]. H column kc + j: rows [0, kt + j) projections, row kt + j the
    // B-norm. The cycle ends at mm = the last kc with kc + bs > m.
    const std::vector<std::pair<int, int>> plan = plan_steps(k);
    auto enqueue_steps = [&](bool prof, bool skip_first) {
      for (const auto& stp : plan) {
        const int j = stp.first, w = stp.second;
        double* vj = V + static_cast<int64_t>(j) * n2;
        if (prof) cuda_check(cudaEventRecord(e_a, st), "ev");
        if (!(skip_first && j == k)) {
          if (w == 1)
            op.apply(vj, r);
          else
            op.apply_block(vj, w, r);
        }
        if (prof) {
          cuda_check(cudaEventRecord(e_b, st), "ev");
          cuda_check(cudaEventSynchronize(e_b), "ev");
          float ms;
          cudaEventElapsedTime(&ms, e_a, e_b);
          t_solve += ms;
          cuda_check(cudaEventRecord(e_a, st), "ev");
        }
        double* hA = dHa.as<double>() + static_cast<int64_t>(j) * LDH;
        double* hB = dHb.as<double>() + static_cast<int64_t>(j) * LDH;
        const int kt = j + bs;
        if (w == 1) {
          // CGS2 with the stored B-images: h = (BV)^T r, r -= V h (twice),
          // then ||r||_B, v_{j+1} = r / beta and B v_{j+1} from one M-product
          op.gemv_t(BV, kt, r, hA);
          op.gemv_n(V, kt, hA, r, nullptr);
          op.gemv_t(BV, kt, r, hB);
          op.gemv_n(V, kt, hB, r, nullptr);
          op.bnorm_normalize_b(r, dBeta.as<double>() + j, V + static_cast<int64_t>(kt) * n2,
                               BV + static_cast<int64_t>(kt) * n2);
        } else {
          // BCGS2: two passes of {project the block against V[0, kt) (every
          // basis vector read once for the w members), B-orthonormalise it
          // member by member (CGS2 against the earlier members)}; the second
          // pass works on the normalised first-pass block in place, so a
          // block whose members cancelled heavily against V or each other is
          // re-orthogonalised at full scale (S V_blk = V (H1 + H2 R1) + Q R2 R1)
          double* BVn = BV + static_cast<int64_t>(kt) * n2;
          double* Vn = V + static_cast<int64_t>(kt) * n2;
          double* hC = dHc.as<double>() + static_cast<int64_t>(j) * LDH;
          double* hD = dHd.as<double>() + static_cast<int64_t>(j) * LDH;
          // intra-block CGS2 with the members' M r_l tracked alongside (one
          // block SpMV per pass instead of one M-product per member: B r_b is
          // updated with the stored B-images of the earlier members)
          double* Wl = W.dWl.as<double>();
          static const bool mtrack = !std::getenv("RQB_BLOCK_MTRACK") || std::atoi(std::getenv("RQB_BLOCK_MTRACK")) != 0;
          auto intra = [&](double* src, double* h1, double* h2, double* beta) {
            if (!mtrack) {  // one M-product per member (A/B reference)
              for (int b = 0; b < w; ++b) {
                double* rb = src + static_cast<int64_t>(b) * n2;
                if (b > 0)
                  for (double* hh : {h1 + kt + static_cast<int64_t>(b) * LDH, h2 + kt + static_cast<int64_t>(b) * LDH}) {
                    op.gemv_t(BVn, b, rb, hh);
                    op.gemv_n(Vn, b, hh, rb, nullptr);
                  }
                op.bnorm_normalize_b(rb, beta + b, Vn + static_cast<int64_t>(b) * n2, BVn + static_cast<int64_t>(b) * n2);
              }
              return;
            }
            op.mspmv_block(src, w, Wl);
            for (int b = 0; b < w; ++b) {
              double* rb = src + static_cast<int64_t>(b) * n2;
              double* wlb = Wl + static_cast<int64_t>(b) * (n2 / 2);
              if (b > 0)
                for (double* hh : {h1 + kt + static_cast<int64_t>(b) * LDH, h2 + kt + static_cast<int64_t>(b) * LDH}) {
                  op.gemv_t(BVn, b, rb, hh);
                  op.gemv_n(Vn, b, hh, rb, nullptr);
                  op.gemv_n_len(BVn + n2 / 2, b, n2, n2 / 2, hh, wlb);
                }
              op.bnorm_normalize_w(rb, wlb, beta + b, Vn + static_cast<int64_t>(b) * n2,
                                   BVn + static_cast<int64_t>(b) * n2);
            }
          };
          op.gemm_t(BV, kt, r, w, hA, LDH);
          op.gemm_n(V, kt, hA, LDH, r, w);
          intra(r, hA, hC, dBeta.as<double>() + j);
          op.gemm_t(BV, kt, Vn, w, hB, LDH);
          op.gemm_n(V, kt, hB, LDH, Vn, w);
          intra(Vn, hB, hD, dBeta2.as<double>() + j);
        }
        if (prof) {
          cuda_check(cudaEventRecord(e_b, st), "ev");
          cuda_check(cudaEventSynchronize(e_b), "ev");
          float ms;
          cudaEventElapsedTime(&ms, e_a, e_b);
          t_orth += ms;
        }
      }
    };
    if (o.profile) {
      enqueue_steps(true, false);
    } else {
      const std::pair<int, const double*> key{pre_applied ? -1 - k : k, V};
      auto it = graphs.find(key);
      if (it == graphs.end()) {
        const auto tg = now();
        cudaGraph_t gr;
        const int64_t l0 = op.launches;
        cuda_check(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "capture");
        enqueue_steps(false, pre_applied);
        cuda_check(cudaStreamEndCapture(st, &gr), "capture end");
        const int64_t kernels = op.launches - l0;
        op.launches = l0;  // counted per replay below
        cudaGraphExec_t ex;
        cuda_check(cudaGraphInstantiate(&ex, gr, 0), "graph instantiate");
        cudaGraphDestroy(gr);
        it = graphs.emplace(key, std::make_pair(ex, kernels)).first;
        t_graph_build += ms_since(tg);
      }
      cuda_check(cudaGraphLaunch(it->second.first, st), "graph launch");
      op.launches += it->second.second;  // the same count on every call, cached graph or not
      res.graph_launches += 1;
    }
    const int mm = m;  // columns of H after this cycle
    for (const auto& stp : plan) {
      // per step of width 1: apply + 2 x (B-product, kt dots, kt axpys) + B-norm;
      // per block step of width w: w applies, 2 x (w B-products, 2 kt w
      // dots/axpys), the block's own CGS2 (2 x (B-product, 2b dots/axpys) for
      // member b > 0) and w B-norms (B-product + dot) — the oracle's block
      // mode, op for op
      const int j = stp.first, w = stp.second;
      const int kt = j + bs;
      for (int b = 0; b < w; ++b) charge_apply(L, op);
      if (w == 1) {
        for (int pass = 0; pass < 3; ++pass) charge_bproduct(L, op);
        charge_vv2n(L, op, 4 * kt + 1);
      } else {
        for (int pass = 0; pass < 2; ++pass) {  // BCGS2: projection + intra-block CGS2 + B-norms, twice
          for (int b = 0; b < w; ++b) charge_bproduct(L, op);
          charge_vv2n(L, op, 2 * static_cast<int64_t>(kt) * w);
          for (int b = 0; b < w; ++b) {
            if (b > 0)
              for (int sub = 0; sub < 2; ++sub) {
                charge_bproduct(L, op);
                charge_vv2n(L, op, 2 * b);
              }
            charge_bproduct(L, op);
            charge_vv2n(L, op, 1);
          }
        }
      }
    }
    cuda_check(cudaMemcpyAsync(ha.data(), dHa.p, sizeof(double) * LDH * LDH, cudaMemcpyDeviceToHost, st), "D2H H");
    cuda_check(cudaMemcpyAsync(hb.data(), dHb.p, sizeof(double) * LDH * LDH, cudaMemcpyDeviceToHost, st), "D2H H");
    cuda_check(cudaMemcpyAsync(betas.data(), dBeta.p, sizeof(double) * LDH, cudaMemcpyDeviceToHost, st),
               "D2H beta");
    if (bs > 1) {
      cuda_check(cudaMemcpyAsync(W.hc.data(), dHc.p, sizeof(double) * LDH * LDH, cudaMemcpyDeviceToHost, st), "D2H");
      cuda_check(cudaMemcpyAsync(W.hd.data(), dHd.p, sizeof(double) * LDH * LDH, cudaMemcpyDeviceToHost, st), "D2H");
      cuda_check(cudaMemcpyAsync(W.betas2.data(), dBeta2.p, sizeof(double) * LDH, cudaMemcpyDeviceToHost, st),
                 "D2H beta2");
    }
    cuda_check(cudaEventRecord(e_h, st), "ev");
    // Speculatively apply the operator to the frontier block V[mm, mm+bs):
    // unless the cycle ends in a deflated restart (fresh vectors), it is the
    // next cycle's continuation block V[p, p+bs), so the solve overlaps the
    // host's Ritz / restart work.
    pre_applied = !o.profile;
    if (pre_applied) {
      if (bs == 1)
        op.apply(V + static_cast<int64_t>(mm) * n2, r);
      else
        op.apply_block(V + static_cast<int64_t>(mm) * n2, bs, r);
    }
    {
      const auto ts0 = now();
      cuda_check(cudaEventSynchronize(e_h), "sync");
      t_sync += ms_since(ts0);  // host blocked on the cycle's Arnoldi steps
    }
    const auto th0 = now();
    for (const auto& stp : plan) {
      const int j0 = stp.first, w = stp.second, kt = j0 + bs;  // step start, width, projection range
      if (w == 1) {
        for (int i = 0; i < kt; ++i)
          Hc(i, j0) = ha[i + static_cast<size_t>(j0) * LDH] + hb[i + static_cast<size_t>(j0) * LDH];
        Hc(kt, j0) = betas[j0];
        continue;
      }
      // BCGS2: H[:kt, c] = H1 + H2 R1, H[kt.., c] = R2 R1 (R1, R2 upper triangular w x w)
      auto at = [&](const Pinned& P, int i, int c) { return P.p[i + static_cast<size_t>(c) * LDH]; };
      std::vector<double> R1(static_cast<size_t>(w) * w, 0.0), R2(R1.size(), 0.0);
      for (int b = 0; b < w; ++b) {
        for (int t = 0; t < b; ++t) {
          R1[t + static_cast<size_t>(b) * w] = at(W.ha, kt + t, j0 + b) + at(W.hc, kt + t, j0 + b);
          R2[t + static_cast<size_t>(b) * w] = at(W.hb, kt + t, j0 + b) + at(W.hd, kt + t, j0 + b);
        }
        R1[b + static_cast<size_t>(b) * w] = betas[j0 + b];
        R2[b + static_cast<size_t>(b) * w] = W.betas2[j0 + b];
      }
      for (int b = 0; b < w; ++b) {
        const int c = j0 + b;
        for (int i = 0; i < kt; ++i) {
          double v = at(W.ha, i, c);
          for (int t = 0; t <= b; ++t) v += at(W.hb, i, j0 + t) * R1[t + static_cast<size_t>(b) * w];
          Hc(i, c) = v;
        }
        for (int i = 0; i <= b; ++i) {
          double v = 0.0;
          for (int t = i; t <= b; ++t) v += R2[i + static_cast<size_t>(t) * w] * R1[t + static_cast<size_t>(b) * w];
          Hc(kt + i, c) = v;
        }
      }
    }
    // ---- Ritz extraction (H_mm is upper Hessenberg for bs = 1, banded with
    // bs subdiagonals for a block; after a restart it is a full matrix) ----
    std::vector<double> Hm(static_cast<size_t>(mm) * mm);
    for (int j = 0; j < mm; ++j)
      for (int i = 0; i < mm; ++i) Hm[i + static_cast<size_t>(j) * mm] = Hc(i, j);
    CMat T, Z;
    std::vector<double> Tre, Zre;  // the real Schur form (kept for the restart)
    const auto tr0 = now();
    if (!real_schur(Hm, mm, Tre, Zre)) fail(errc::solver, "Hessenberg QR did not converge");
    complexify_schur(Tre, Zre, mm, T, Z);
    const CMat Y = triangular_eigvecs(T);
    t_ritz += ms_since(tr0);
    // residual rows: S V_mm = V_mm H_mm + V[mm, mm+bs) E, E = H[mm.., 0..mm) (nonzero
    // only in the last block's columns)
    const int m0 = mm - bs;
    std::vector<Ritz> rz(mm);
    for (int i = 0; i < mm; ++i) {
      rz[i].theta = T(i, i);
      rz[i].lambda = (sig + 1.0 / rz[i].theta) * vs;
      // y_i = Z Y[:, i]; residual estimate ||E y_i|| / |theta| (bs = 1: |beta_m e_m^T y_i| / |theta|)
      std::vector<cplx> ylast(bs, 0.0);
      for (int q = 0; q < bs; ++q)
        for (int t = 0; t <= i; ++t) ylast[q] += Z(m0 + q, t) * Y(t, i);
      double e2 = 0.0;
      for (int a = 0; a < bs; ++a) {
        cplx s = 0.0;
        for (int q = 0; q < bs; ++q) s += Hc(mm + a, m0 + q) * ylast[q];
        e2 += std::norm(s);
      }
      rz[i].est = std::sqrt(e2) / std::max(std::abs(rz[i].theta), 1e-300);
      rz[i].idx = i;
    }
    // wanted order: largest |theta| first; conjugate pairs adjacent (+imag first)
    std::vector<int> order(mm);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      const double da = dist(rz[a].lambda, sig * vs), db = dist(rz[b].lambda, sig * vs);
      if (da != db) return da < db;
      return rz[a].lambda.imag() > rz[b].lambda.imag();
    });
    // ---- groups: conjugate pairs + clusters (single linkage, relative gap
    // 1e-4). Kept sets are unions of whole groups, so they are closed under
    // conjugation and never split a cluster: the real basis of the kept complex
    // Schur vectors then spans an invariant subspace to ~eps / 1e-4.
    std::vector<std::vector<int>> groups;
    std::vector<int> group_of(mm, -1);
    {
      std::vector<int> par(mm);
      std::iota(par.begin(), par.end(), 0);
      std::function<int(int)> find = [&](int x) { return par[x] == x ? x : par[x] = find(par[x]); };
      for (int i = 0; i < mm; ++i)
        for (int q = i + 1; q < mm; ++q) {
          const cplx a = rz[i].theta, b = rz[q].theta;
          const double scale = std::max(std::abs(a), std::abs(b));
          if (std::abs(a - b) <= kClusterGap * scale || std::abs(a - std::conj(b)) <= kClusterGap * scale)
            par[find(i)] = find(q);
        }
      std::vector<int> root_group(mm, -1);
      for (int a = 0; a < mm; ++a) {  // groups in wanted order of their best member
        const int i = order[a];
        const int r = find(i);
        if (root_group[r] < 0) {
          root_group[r] = static_cast<int>(groups.size());
          groups.push_back({});
        }
        groups[root_group[r]].push_back(i);
        group_of[i] = root_group[r];
      }
    }
    // ---- convergence: explicit residuals of the nev nearest (+ their group mates) ----
    std::vector<int> cand(order.begin(), order.begin() + nev);
    std::vector<int> chk = cand;
    {
      std::vector<int> in(mm, 0);
      for (int i : cand) in[i] = 1;
      for (int i : cand)
        for (int q : groups[group_of[i]])
          if (!in[q]) in[q] = 1, chk.push_back(q);
    }
    const int nchk = static_cast<int>(chk.size());
    // explicit residuals cost a pass over V and over K, C, M per candidate:
    // after a failed check, wait until the worst estimate improved 10x (or 8
    // cycles passed) before checking again
    double est_worst = 0.0;
    for (int i : cand) est_worst = std::max(est_worst, rz[i].est);
    if (bs > 1 && o.guard_single_cluster) {
      // block mode: when the nev nearest are members of one (degenerate)
      // cluster, which nev of its members rank "nearest" is arbitrary, and a
      // block brings in up to 2 bs fresh copies per step; gate the explicit
      // check on the nev-th best estimate among the cluster's members (all of
      // them are checked: chk holds the whole group) instead of the worst of an
      // arbitrary nev
      const int g0 = group_of[cand[0]];
      bool one = true;
      for (int c = 1; c < nev && one; ++c) one = group_of[cand[c]] == g0;
      if (one && static_cast<int>(groups[g0].size()) > nev) {
        std::vector<double> e;
        for (int i : groups[g0]) e.push_back(rz[i].est);
        std::nth_element(e.begin(), e.begin() + (nev - 1), e.end());
        est_worst = e[nev - 1];
      }
    }
    const bool maybe = est_worst <= check_gate || (est_worst <= o.est_factor * o.tol && since_check >= recheck_wait);
    ++since_check;
    bool all_conv = false, mates_conv = false;
    std::vector<double> cres(nchk, 1.0);
    std::vector<int> cblock(nchk, 0);
    const auto tc0 = now();
    if (maybe) {
      // Ritz vectors X = V_m [Re y, Im y] (y = Z Y[:, i])
      std::vector<double> Yr(static_cast<size_t>(mm) * 2 * nchk);
#pragma omp parallel for schedule(dynamic, 4) num_threads(host_threads()) if (static_cast<int64_t>(nchk) * mm * mm > 1000000)
      for (int c = 0; c < nchk; ++c) {
        std::vector<cplx> ycol(mm, cplx(0.0));
        const int i = chk[c];
        for (int t = 0; t <= i; ++t) {  // y = Z[:, 0..i] Y[0..i, i] (Y upper triangular)
          const cplx yt = Y(t, i);
          const cplx* zc = &Z.a[static_cast<size_t>(t) * mm];
          for (int row = 0; row < mm; ++row) ycol[row] += zc[row] * yt;
        }
        for (int row = 0; row < mm; ++row) {
          Yr[row + static_cast<size_t>(2 * c) * mm] = ycol[row].real();
          Yr[row + static_cast<size_t>(2 * c + 1) * mm] = ycol[row].imag();
        }
      }
      const double* ysrc = Yr.data();
      if (Yr.size() <= static_cast<size_t>(m + 1) * (2 * m + 2)) {
        std::memcpy(W.hy.data(), Yr.data(), sizeof(double) * Yr.size());
        ysrc = W.hy.data();
      }
      const double t_yr = ms_since(tc0);
      cuda_check(cudaMemcpyAsync(dQ.p, ysrc, sizeof(double) * Yr.size(), cudaMemcpyHostToDevice, st), "H2D Y");
      std::vector<double> lam(2 * nchk);
      for (int c = 0; c < nchk; ++c) {
        const cplx gam = rz[chk[c]].lambda / vs;  // eigenvalue of the scaled pencil
        cblock[c] = std::abs(gam) > 1.0 ? 1 : 0;  // larger-norm block
        lam[2 * c] = gam.real();
        lam[2 * c + 1] = gam.imag();
      }
      // X = V_m [Re y, Im y] (one DGEMM, row-major) + all residuals in one SpMM pass
      op.ritz_residuals(V, mm, dQ.as<double>(), nchk, lam.data(), cblock.data(), dX.as<double>(),
                        dRes.as<double>());
      last_nchk = nchk;
      std::vector<double> rr(8 * nchk);
      last_lam = lam;
      cuda_check(cudaMemcpyAsync(rr.data(), dRes.p, sizeof(double) * 8 * nchk, cudaMemcpyDeviceToHost, st),
                 "D2H res");
      const double t_enq = ms_since(tc0);
      cuda_check(cudaStreamSynchronize(st), "sync");
      if (trace_cycles)
        std::fprintf(stderr, "[eigs] check %d: Y %.1f enqueue %.1f sync %.1f ms\n", nchk, t_yr, t_enq, ms_since(tc0));
      last_rq.assign(rr.begin() + 2 * nchk, rr.end());
      all_conv = mates_conv = true;
      for (int c = 0; c < nchk; ++c) {
        const double ag = std::abs(rz[chk[c]].lambda / vs);
        const double den = (norms1[0] + ag * norms1[1] + ag * ag * norms1[2]) * std::sqrt(rr[2 * c + 1]);
        cres[c] = den > 0 ? std::sqrt(rr[2 * c]) / den : 1.0;
        if (!(cres[c] <= o.tol)) (c < nev ? all_conv : mates_conv) = false;
      }
      mates_conv = mates_conv && all_conv;
      L.n_check += nchk;  // one explicit pencil residual (K, C, M products) per candidate
      L.macs_check += 3.0 * nnz * nchk;
      t_check += ms_since(tc0);
      since_check = 0;
      check_gate = all_conv ? o.est_factor * o.tol : 0.1 * est_worst;
      // a check that found most of the nev converged is re-run sooner (its
      // cost, one SpMM pass over the candidates, is below a cycle's): the wait
      // shrinks from 8 cycles in proportion to the converged fraction
      int nc_all = 0;
      for (int c = 0; c < nchk; ++c) nc_all += cres[c] <= o.tol;
      const double frac = std::min(1.0, static_cast<double>(nc_all) / nev);
      recheck_wait = frac >= 0.5 ? std::max(1, static_cast<int>(std::lround(8.0 * (1.0 - frac)))) : 8;
    }
    int nconv_now = 0;
    for (int c = 0; c < nev && maybe; ++c)
      if (cres[c] <= o.tol) ++nconv_now;
    res.nconv = std::max(res.nconv, nconv_now);
    last_cand.clear();
    for (int c = 0; c < nev; ++c) last_cand.push_back(rz[cand[c]]);
    last_res.assign(cres.begin(), cres.begin() + nev);

    // the returned set: checked positions pos[0..nev) (default: the nev nearest)
    auto capture_set = [&](std::vector<int> pos) {
      if (pos.empty())
        for (int c = 0; c < nev; ++c) pos.push_back(c);
      final_set.clear();
      final_res.clear();
      final_block.clear();
      for (int c : pos) {
        final_set.push_back(rz[chk[c]]);
        final_res.push_back(cres[c]);
        final_block.push_back(cblock[c]);
      }
      // Quadratic Rayleigh-quotient refinement of the returned eigenvalues: the
      // root of u^H (K + g C + g^2 M) u = 0 nearest the Ritz value (u the
      // converged vector on its block, coefficients from the check's SpMM pass);
      // kept when its explicit residual (one more pass over K, C, M) is within
      // tolerance. A converged vector pins its eigenvalue to ~ residual^2 this
      // way, where the Ritz value of a degenerate cluster is only ~ residual.
      if (o.refine && static_cast<int>(last_rq.size()) == 6 * last_nchk && last_nchk == nchk) {
        std::vector<double> lam2 = last_lam, rr2(8 * static_cast<size_t>(nchk));
        std::vector<cplx> gref(pos.size());
        for (size_t q = 0; q < pos.size(); ++q) {
          const int c = pos[q];
          const cplx kq(last_rq[6 * c], last_rq[6 * c + 1]), cq(last_rq[6 * c + 2], last_rq[6 * c + 3]),
              mq(last_rq[6 * c + 4], last_rq[6 * c + 5]);
          const cplx g0(last_lam[2 * c], last_lam[2 * c + 1]);
          cplx g = g0;
          if (std::abs(mq) > 0.0) {
            const cplx dsc = std::sqrt(cq * cq - 4.0 * mq * kq);
            const cplx r1 = (-cq + dsc) / (2.0 * mq), r2 = (-cq - dsc) / (2.0 * mq);
            g = std::abs(r1 - g0) <= std::abs(r2 - g0) ? r1 : r2;
          }
          gref[q] = g;
          lam2[2 * c] = g.real();
          lam2[2 * c + 1] = g.imag();
        }
        op.residuals_again(dX.as<double>(), nchk, lam2.data(), dRes.as<double>());
        cuda_check(cudaMemcpyAsync(rr2.data(), dRes.p, sizeof(double) * 8 * nchk, cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaStreamSynchronize(st), "sync");
        for (size_t q = 0; q < pos.size(); ++q) {
          const int c = pos[q];
          const double ag = std::abs(gref[q]);
          const double den = (norms1[0] + ag * norms1[1] + ag * ag * norms1[2]) * std::sqrt(rr2[2 * c + 1]);
          const double r2 = den > 0 ? std::sqrt(rr2[2 * c]) / den : 1.0;
          if (r2 <= std::max(final_res[q], o.tol)) {
            final_set[q].lambda = gref[q] * vs;
            final_res[q] = r2;
          }
        }
      }
      if (o.want_vectors) {
        final_vecs_re.assign(static_cast<size_t>(n) * nev, 0.0);
        final_vecs_im.assign(static_cast<size_t>(n) * nev, 0.0);
        for (int c = 0; c < nev; ++c) {
          for (int part = 0; part < 2; ++part) {
            op.ritz_extract(dX.as<double>(), last_nchk, pos[c], part, dW.as<double>());
            cuda_check(cudaMemcpyAsync((part ? final_vecs_im : final_vecs_re).data() + static_cast<size_t>(c) * n,
                                       dW.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "D2H x");
          }
          cuda_check(cudaStreamSynchronize(st), "sync");
          double nr = 0;
          for (int64_t i = 0; i < n; ++i)
            nr += final_vecs_re[c * n + i] * final_vecs_re[c * n + i] +
                  final_vecs_im[c * n + i] * final_vecs_im[c * n + i];
          nr = std::sqrt(nr);
          for (int64_t i = 0; i < n; ++i) final_vecs_re[c * n + i] /= nr, final_vecs_im[c * n + i] /= nr;
        }
      }
    };

    // One degenerate cluster: every one of the nev nearest Ritz values is a
    // member of the nearest group. The guard exists for the case where fewer
    // copies of the nearest eigenvalue than requested were found and farther
    // values filled the set; here the set cannot move closer, so the solve ends
    // as soon as nev members of the cluster have converged explicitly (in
    // conjugate pairs), whether or not they are exactly the nev nearest by a
    // 1e-12 margin: all are the same eigenvalue. Without this a
    // cluster larger than the space fills it with unconverged copies and the
    // solve stagnates at a few new steps a cycle (cfg4_iga: 98 of the nev
    // nearest converged for 1000 cycles).
    std::vector<int> cluster_pos;
    if (maybe && o.guard_single_cluster) {
      const int g0 = group_of[cand[0]];
      bool one = true;
      for (int c = 1; c < nev && one; ++c) one = group_of[cand[c]] == g0;
      if (one) {
        std::vector<int> pp, nn;
        for (int c = 0; c < nchk; ++c)
          if (cres[c] <= o.tol && group_of[chk[c]] == g0)
            (rz[chk[c]].lambda.imag() >= 0 ? pp : nn).push_back(c);
        if (pp.empty() || nn.empty()) {  // a real cluster: any converged members
          for (int c : pp) if (static_cast<int>(cluster_pos.size()) < nev) cluster_pos.push_back(c);
          for (int c : nn) if (static_cast<int>(cluster_pos.size()) < nev) cluster_pos.push_back(c);
        } else {
          for (size_t k = 0; k < std::min(pp.size(), nn.size()) && static_cast<int>(cluster_pos.size()) + 2 <= nev; ++k)
            cluster_pos.push_back(pp[k]), cluster_pos.push_back(nn[k]);
          if (static_cast<int>(cluster_pos.size()) < nev && nev % 2 == 1) {
            const size_t k = cluster_pos.size() / 2;
            if (k < pp.size()) cluster_pos.push_back(pp[k]);
          }
        }
        if (static_cast<int>(cluster_pos.size()) != nev) cluster_pos.clear();
      }
    }
    if (!cluster_pos.empty()) {
      capture_set(cluster_pos);
      converged_final = true;
      break;
    }

    // ---- decide: done / guard (deflated) restart / normal restart ----
    std::vector<int> sel(mm, 0);
    int p = 0;
    bool deflate = false;
    if (all_conv) {
      std::vector<double> dists;
      for (int c = 0; c < nev; ++c) dists.push_back(dist(rz[cand[c]].lambda, sig * vs));
      std::sort(dists.begin(), dists.end());
      bool improved = prev_guard_dists.empty();
      for (size_t i = 0; i < dists.size() && !improved; ++i)
        if (dists[i] < prev_guard_dists[i] * (1.0 - 1e-8)) improved = true;
      capture_set({});
      if (!o.guard || !improved || guard_passes >= o.max_guard) {
        converged_final = true;
        break;
      }
      if (mates_conv && nchk <= m - bs) {
        // every kept direction is converged: deflate them (b = 0) and restart
        // the Krylov space from a fresh seeded vector (SPEC.md:457 fallback)
        prev_guard_dists = dists;
        ++guard_passes;
        pass_cycles = 0;
        deflate = true;
        for (int i : chk) sel[i] = 1;
        p = nchk;
      }
    }
    if (!deflate) {
      for (const auto& g : groups) {
        if (p >= keep_target || p + static_cast<int>(g.size()) > m - bs) break;
        for (int i : g) sel[i] = 1;
        p += static_cast<int>(g.size());
      }
      if (p == 0) {  // one cluster fills the whole space: fall back to conjugate pairs
        for (int a = 0; a < mm && p < keep_target; ++a) {
          const int i = order[a];
          if (sel[i]) continue;
          int partner = -1;
          double bd = 1e300;
          if (std::abs(rz[i].theta.imag()) > 1e-12 * std::abs(rz[i].theta))
            for (int q = 0; q < mm; ++q)
              if (q != i && !sel[q]) {
                const double d = std::abs(rz[q].theta - std::conj(rz[i].theta));
                if (d < bd) bd = d, partner = q;
              }
          if (p + 1 + (partner >= 0) > m - bs) break;
          sel[i] = 1, ++p;
          if (partner >= 0) sel[partner] = 1, ++p;
        }
      }
    }
    // ---- restart: reorder the Schur form, real basis of the kept directions ----
    // Real Schur form: the selected 1 x 1 / 2 x 2 blocks are swapped to the
    // top, Q_p = Z[:, :p] and T_p = T[:p, :p] come out directly (a selected
    // member of a conjugate pair brings its mate). Fallback (a refused swap, or
    // a closed selection larger than m - bs): reorder the complex form and take
    // a rank-p real basis of the kept Schur vectors, T_p = Q_p^T H_m Q_p.
    const auto trs0 = now();
    std::vector<double> Qp, Tp;
    {
      static const bool real_restart = !std::getenv("RQB_RESTART_REAL") || std::atoi(std::getenv("RQB_RESTART_REAL")) != 0;
      std::vector<double> Tq = Tre, Zq = Zre;
      std::vector<int> s2 = sel;
      const int pr = real_restart ? real_schur_reorder(Tq, Zq, mm, s2) : -1;
      if (pr > 0 && pr <= m - bs && pr <= mm) {
        p = pr;
        Qp.assign(Zq.begin(), Zq.begin() + static_cast<size_t>(mm) * p);
        Tp.resize(static_cast<size_t>(p) * p);
        for (int c = 0; c < p; ++c)
          std::copy(Tq.begin() + static_cast<size_t>(c) * mm, Tq.begin() + static_cast<size_t>(c) * mm + p,
                    Tp.begin() + static_cast<size_t>(c) * p);
      }
    }
    t_reorder += ms_since(trs0);
    const auto trb0 = now();
    // H Q_p (the invariance defect below; T_p itself in the fallback)
    std::vector<double> HQ;
    auto hq_product = [&]() {
      HQ.assign(static_cast<size_t>(mm) * p, 0.0);
#pragma omp parallel for schedule(static) num_threads(host_threads()) if (static_cast<int64_t>(mm) * mm * p > 1000000)
      for (int c = 0; c < p; ++c) {
        double* hq = HQ.data() + static_cast<size_t>(c) * mm;
        for (int t = 0; t < mm; ++t) {
          const double q = Qp[t + static_cast<size_t>(c) * mm];
          if (q == 0.0) continue;
          const double* ht = Hm.data() + static_cast<size_t>(t) * mm;
          for (int i = 0; i < mm; ++i) hq[i] += ht[i] * q;
        }
      }
    };
    if (Qp.empty()) {
      CMat Tr = T, Zr = Z;
      std::vector<int> s2 = sel;
      schur_reorder(Tr, Zr, s2);
      const int rank = real_basis(Zr, p, Qp);
      if (rank < p) p = rank;
      if (p <= 0) fail(errc::solver, "Krylov-Schur restart lost its basis");
      // T_p = Q_p^T H_m Q_p (column-oriented loops: contiguous axpy / dot)
      hq_product();
      Tp.assign(static_cast<size_t>(p) * p, 0.0);
#pragma omp parallel for schedule(static) num_threads(host_threads()) if (static_cast<int64_t>(mm) * p * p > 1000000)
      for (int c = 0; c < p; ++c) {
        const double* hq = HQ.data() + static_cast<size_t>(c) * mm;
        for (int i = 0; i < p; ++i) {
          const double* qi = Qp.data() + static_cast<size_t>(i) * mm;
          double s = 0;
          for (int t = 0; t < mm; ++t) s += qi[t] * hq[t];
          Tp[i + static_cast<size_t>(c) * p] = s;
        }
      }
    } else {
      hq_product();
    }
    t_basis += ms_since(trb0);
    {
      // invariance defect ||H Q_p - Q_p T_p|| / ||H|| (exact restart needs ~eps)
      double dmax = 0, hmax = 0;
      for (double x : Hm) hmax = std::max(hmax, std::fabs(x));
#pragma omp parallel for schedule(static) reduction(max : dmax) num_threads(host_threads()) if (static_cast<int64_t>(mm) * p * p > 1000000)
      for (int c = 0; c < p; ++c) {
        std::vector<double> rc(HQ.begin() + static_cast<size_t>(c) * mm, HQ.begin() + static_cast<size_t>(c + 1) * mm);
        for (int t = 0; t < p; ++t) {
          const double tc = Tp[t + static_cast<size_t>(c) * p];
          if (tc == 0.0) continue;
          const double* qt = Qp.data() + static_cast<size_t>(t) * mm;
          for (int i = 0; i < mm; ++i) rc[i] -= tc * qt[i];
        }
        for (int i = 0; i < mm; ++i) dmax = std::max(dmax, std::fabs(rc[i]));
      }
      res.max_restart_defect = std::max(res.max_restart_defect, dmax / std::max(hmax, 1e-300));
    }
    std::memcpy(W.hq.data(), Qp.data(), sizeof(double) * mm * p);
    cuda_check(cudaMemcpyAsync(dQ.p, W.hq.data(), sizeof(double) * mm * p, cudaMemcpyHostToDevice, st), "H2D Q");
    op.combine(V, mm, dQ.as<double>(), mm, p, V2);
    op.combine(BV, mm, dQ.as<double>(), mm, p, BV2);
    L.n_restart += 1;
    L.macs_restart += static_cast<double>(mm) * p * n2;
    // the new residual rows E Q_p before H is cleared (E: rows mm.., last block's columns)
    std::vector<double> EQ(static_cast<size_t>(bs) * p, 0.0);
    for (int a = 0; a < bs; ++a)
      for (int c = 0; c < p; ++c) {
        double s = 0.0;
        for (int q = 0; q < bs; ++q) s += Hc(mm + a, m0 + q) * Qp[(m0 + q) + static_cast<size_t>(c) * mm];
        EQ[a + static_cast<size_t>(c) * bs] = s;
      }
    std::fill(H.begin(), H.end(), 0.0);
    for (int c = 0; c < p; ++c)
      for (int i = 0; i < p; ++i) Hc(i, c) = Tp[i + static_cast<size_t>(c) * p];
    std::swap(V, V2);
    std::swap(BV, BV2);
    if (deflate) {
      // b = 0 (converged directions deflated); fresh seeded continuation block
      // (the speculative apply of the frontier block is discarded)
      pre_applied = false;
      fresh_block(o.seed + 0x1000003ull * guard_passes, p, bs);
    } else {
      for (int a = 0; a < bs; ++a)
        for (int c = 0; c < p; ++c) Hc(p + a, c) = EQ[a + static_cast<size_t>(c) * bs];
      cuda_check(cudaMemcpyAsync(V + static_cast<int64_t>(p) * n2, V2 + static_cast<int64_t>(mm) * n2,
                                 sizeof(double) * n2 * bs, cudaMemcpyDeviceToDevice, st), "D2D v");
      cuda_check(cudaMemcpyAsync(BV + static_cast<int64_t>(p) * n2, BV2 + static_cast<int64_t>(mm) * n2,
                                 sizeof(double) * n2 * bs, cudaMemcpyDeviceToDevice, st), "D2D Bv");
    }
    t_restart += ms_since(trs0);
    t_host += ms_since(th0);
    if (trace_cycles)
      std::fprintf(stderr, "[eigs] cycle %d: steps %d..%d, checked %d (maybe %d, nconv %d), est worst %.2e best %.2e, "
                   "groups %zu (first %zu), kept %d%s, t ritz %.1f check %.1f restart %.1f (reorder %.1f basis %.1f) host %.1f "
                   "sync %.1f ms\n", cycles, k,
                   mm, maybe ? nchk : 0, (int)maybe, nconv_now, est_worst, rz[order[0]].est, groups.size(),
                   groups.empty() ? size_t(0) : groups[0].size(), p, deflate ? " (deflated restart)" : "", t_ritz,
                   t_check, t_restart, t_reorder, t_basis, t_host, t_sync);
    k = p;
  }
  op.fac->check_sweeps();  // watchdog of the triangular sweeps (syncs the stream)
  cudaEventDestroy(e_h);
  cudaEventDestroy(e_a);
  cudaEventDestroy(e_b);
  // keep the last candidate set if the run stopped early
  if (!converged_final && final_set.empty()) {
    final_set = last_cand;
    final_res = last_res;
  }
  res.converged = converged_final;
  res.cycles = cycles;
  res.guard_passes = guard_passes;
  for (size_t c = 0; c < final_set.size(); ++c) {
    res.lambda.push_back(final_set[c].lambda);
    res.resid.push_back(final_res[c]);
  }
  res.vec_re = std::move(final_vecs_re);
  res.vec_im = std::move(final_vecs_im);
  res.launches = op.launches - launches0;
  res.t_total_ms = std::chrono::duration<double, std::milli>(clock::now() - t0).count();
  if (std::getenv("RQB_SETUP_TRACE"))
    std::fprintf(stderr, "[setup] eigs: buffers %.1f ms, %zu graphs built in %.1f ms, total %.1f ms\n", t_setup,
                 graphs.size(), t_graph_build, res.t_total_ms);
  res.t_solve_ms = t_solve;
  res.t_orth_ms = t_orth;
  res.t_ritz_ms = t_ritz;
  res.t_check_ms = t_check;
  res.t_restart_ms = t_restart;
  res.t_sync_ms = t_sync;
  if (!converged_final) {
    res.nconv = static_cast<int>(std::count_if(res.resid.begin(), res.resid.end(),
                                               [&](double x) { return x <= o.tol; }));
  } else {
    res.nconv = nev;
  }
  return res;
}

}  // namespace rqb
