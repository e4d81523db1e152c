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
  int m = -1;
  int64_t n2 = 0;
  DeviceBuffer dV, dV2, dBV, dBV2, dR, dW, dHa, dHb, dBeta, dQ, dX, dRes;
  Pinned ha, hb, betas;
  Pinned hv, hq, hy;  // staging of the host -> device copies (start vectors, restart Q, Ritz Y)
  // cycle graph per (start index, basis buffer) and the kernels it launches
  std::map<std::pair<int, const double*>, std::pair<cudaGraphExec_t, int64_t>> graphs;
  EigWorkspace(int m_, int64_t n2_)
      : m(m_), n2(n2_), ha(static_cast<size_t>(m_ + 1) * (m_ + 1)), hb(static_cast<size_t>(m_ + 1) * (m_ + 1)),
        betas(m_ + 1), hv(static_cast<size_t>(n2_)), hq(static_cast<size_t>(m_ + 1) * (2 * m_ + 2)),
        hy(static_cast<size_t>(m_ + 1) * (2 * m_ + 2)) {
    dV.alloc(sizeof(double) * (m + 1) * n2);
    dV2.alloc(sizeof(double) * (m + 1) * n2);
    dBV.alloc(sizeof(double) * (m + 1) * n2);
    dBV2.alloc(sizeof(double) * (m + 1) * n2);
    dR.alloc(sizeof(double) * n2);
    dW.alloc(sizeof(double) * n2);
    dHa.alloc(sizeof(double) * (m + 1) * (m + 1));
    dHb.alloc(sizeof(double) * (m + 1) * (m + 1));
    dBeta.alloc(sizeof(double) * (m + 1));
    dQ.alloc(sizeof(double) * (m + 1) * (2 * m + 2));
    dX.alloc(sizeof(double) * n2 * 2 * (m + 1));
    dRes.alloc(sizeof(double) * 4 * (m + 1));
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
  if (m >= n2) fail(errc::config, "Krylov dimension must be below 2N");
  if (!(o.tol > 0)) fail(errc::config, "tolerance must be positive");
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
  if (!wsp || wsp->m != m || wsp->n2 != n2) {
    op.eig_ws.reset();
    auto fresh = std::make_shared<EigWorkspace>(m, n2);
    wsp = fresh.get();
    op.eig_ws = fresh;
  }
  EigWorkspace& W = *wsp;
  DeviceBuffer &dV = W.dV, &dV2 = W.dV2, &dBV = W.dBV, &dBV2 = W.dBV2, &dR = W.dR, &dW = W.dW, &dHa = W.dHa, &dHb = W.dHb,
               &dBeta = W.dBeta, &dQ = W.dQ, &dX = W.dX, &dRes = W.dRes;
  double* V = dV.as<double>();
  double* V2 = dV2.as<double>();
  double* BV = dBV.as<double>();
  double* BV2 = dBV2.as<double>();
  double* r = dR.as<double>();

  cudaEvent_t e_a, e_b;
  cuda_check(cudaEventCreate(&e_a), "event");
  cuda_check(cudaEventCreate(&e_b), "event");

  // Start vector v = splitmix64(seed) uniform[-1,1]^{2N}, B-normalised.
  auto fresh_vector = [&](uint64_t seed, int nlock, double* dst, double* dst_b) {
    std::vector<double> v(n2);
    uint64_t s = seed;
    for (int64_t i = 0; i < n2; ++i) v[i] = splitmix_uniform(s);
    std::memcpy(W.hv.data(), v.data(), sizeof(double) * n2);
    cuda_check(cudaMemcpyAsync(r, W.hv.data(), sizeof(double) * n2, cudaMemcpyHostToDevice, st), "H2D v0");
    for (int pass = 0; pass < 2 && nlock > 0; ++pass) {
      op.gemv_t(BV, nlock, r, dHa.as<double>());
      op.gemv_n(V, nlock, dHa.as<double>(), r, nullptr);
      charge_bproduct(L, op);  // ledger: the reference algorithm's B-product
      charge_vv2n(L, op, 2 * nlock);
    }
    op.bnorm_normalize_b(r, dBeta.as<double>() + m, dst, dst_b);
    charge_bproduct(L, op);
    charge_vv2n(L, op, 1);
  };

  std::vector<double> H(static_cast<size_t>(m + 1) * m, 0.0);  // column-major (m+1) x m
  auto Hc = [&](int i, int j) -> double& { return H[i + static_cast<size_t>(j) * (m + 1)]; };

  fresh_vector(o.seed, 0, V, BV);
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
  double check_gate = o.est_factor * o.tol;
  int last_nchk = 0;  // candidates of the last explicit check (row-major Ritz batch in dX)
  int since_check = 0;
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
    auto enqueue_steps = [&](bool prof, bool skip_first) {
      for (int j = k; j < m; ++j) {
        double* vj = V + static_cast<int64_t>(j) * n2;
        if (prof) cuda_check(cudaEventRecord(e_a, st), "ev");
        if (!(skip_first && j == k)) op.apply(vj, r);
        if (prof) {
          cuda_check(cudaEventRecord(e_b, st), "ev");
          cuda_check(cudaEventSynchronize(e_b), "ev");
          float ms;
          cudaEventElapsedTime(&ms, e_a, e_b);
          t_solve += ms;
          cuda_check(cudaEventRecord(e_a, st), "ev");
        }
        double* hA = dHa.as<double>() + static_cast<int64_t>(j) * (m + 1);
        double* hB = dHb.as<double>() + static_cast<int64_t>(j) * (m + 1);
        // CGS2 with the stored B-images: h = (BV)^T r, r -= V h (twice),
        // then ||r||_B, v_{j+1} = r / beta and B v_{j+1} from one M-product
        op.gemv_t(BV, j + 1, r, hA);
        op.gemv_n(V, j + 1, hA, r, nullptr);
        op.gemv_t(BV, j + 1, r, hB);
        op.gemv_n(V, j + 1, hB, r, nullptr);
        op.bnorm_normalize_b(r, dBeta.as<double>() + j, V + static_cast<int64_t>(j + 1) * n2,
                             BV + static_cast<int64_t>(j + 1) * n2);
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
    for (int j = k; j < m; ++j) {  // per step: apply + 2 x (B-product, j+1 dots, j+1 axpys) + B-norm
      charge_apply(L, op);
      for (int pass = 0; pass < 3; ++pass) charge_bproduct(L, op);
      charge_vv2n(L, op, 4 * (j + 1) + 1);
    }
    cuda_check(cudaMemcpyAsync(ha.data(), dHa.p, sizeof(double) * (m + 1) * (m + 1),
                               cudaMemcpyDeviceToHost, st), "D2H H");
    cuda_check(cudaMemcpyAsync(hb.data(), dHb.p, sizeof(double) * (m + 1) * (m + 1),
                               cudaMemcpyDeviceToHost, st), "D2H H");
    cuda_check(cudaMemcpyAsync(betas.data(), dBeta.p, sizeof(double) * (m + 1),
                               cudaMemcpyDeviceToHost, st), "D2H beta");
    cuda_check(cudaEventRecord(e_h, st), "ev");
    // Speculatively apply the operator to v_m: unless the cycle ends in a
    // deflated restart (fresh vector), v_m is the next cycle's continuation
    // vector V[p], so the solve overlaps the host's Ritz / restart work.
    pre_applied = !o.profile;
    if (pre_applied) op.apply(V + static_cast<int64_t>(m) * n2, r);
    {
      const auto ts0 = now();
      cuda_check(cudaEventSynchronize(e_h), "sync");
      t_sync += ms_since(ts0);  // host blocked on the cycle's Arnoldi steps
    }
    for (int j = k; j < m; ++j) {
      for (int i = 0; i <= j; ++i)
        Hc(i, j) = ha[i + static_cast<size_t>(j) * (m + 1)] + hb[i + static_cast<size_t>(j) * (m + 1)];
      Hc(j + 1, j) = betas[j];
    }
    // ---- Ritz extraction ----
    std::vector<double> Hm(static_cast<size_t>(m) * m);
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < m; ++i) Hm[i + static_cast<size_t>(j) * m] = Hc(i, j);
    CMat T, Z;
    const auto tr0 = now();
    if (!complex_schur(Hm, m, T, Z)) fail(errc::solver, "Hessenberg QR did not converge");
    const CMat Y = triangular_eigvecs(T);
    t_ritz += ms_since(tr0);
    const double beta_m = Hc(m, m - 1);
    std::vector<Ritz> rz(m);
    for (int i = 0; i < m; ++i) {
      rz[i].theta = T(i, i);
      rz[i].lambda = (sig + 1.0 / rz[i].theta) * vs;
      // y_i in the H basis = Z Y[:, i]; residual estimate |beta_m e_m^T y_i| / |theta|
      cplx ylast = 0.0;
      for (int t = 0; t <= i; ++t) ylast += Z(m - 1, t) * Y(t, i);
      rz[i].est = std::abs(beta_m * ylast) / std::max(std::abs(rz[i].theta), 1e-300);
      rz[i].idx = i;
    }
    // wanted order: largest |theta| first; conjugate pairs adjacent (+imag first)
    std::vector<int> order(m);
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
    std::vector<int> group_of(m, -1);
    {
      std::vector<int> par(m);
      std::iota(par.begin(), par.end(), 0);
      std::function<int(int)> find = [&](int x) { return par[x] == x ? x : par[x] = find(par[x]); };
      for (int i = 0; i < m; ++i)
        for (int q = i + 1; q < m; ++q) {
          const cplx a = rz[i].theta, b = rz[q].theta;
          const double scale = std::max(std::abs(a), std::abs(b));
          if (std::abs(a - b) <= kClusterGap * scale || std::abs(a - std::conj(b)) <= kClusterGap * scale)
            par[find(i)] = find(q);
        }
      std::vector<int> root_group(m, -1);
      for (int a = 0; a < m; ++a) {  // groups in wanted order of their best member
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
      std::vector<int> in(m, 0);
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
    const bool maybe = est_worst <= check_gate || (est_worst <= o.est_factor * o.tol && since_check >= 8);
    ++since_check;
    bool all_conv = false, mates_conv = false;
    std::vector<double> cres(nchk, 1.0);
    std::vector<int> cblock(nchk, 0);
    const auto tc0 = now();
    if (maybe) {
      // Ritz vectors X = V_m [Re y, Im y] (y = Z Y[:, i])
      std::vector<double> Yr(static_cast<size_t>(m) * 2 * nchk);
      std::vector<cplx> ycol(m);
      for (int c = 0; c < nchk; ++c) {
        const int i = chk[c];
        std::fill(ycol.begin(), ycol.end(), cplx(0.0));
        for (int t = 0; t <= i; ++t) {  // y = Z[:, 0..i] Y[0..i, i] (Y upper triangular)
          const cplx yt = Y(t, i);
          const cplx* zc = &Z.a[static_cast<size_t>(t) * m];
          for (int row = 0; row < m; ++row) ycol[row] += zc[row] * yt;
        }
        for (int row = 0; row < m; ++row) {
          Yr[row + static_cast<size_t>(2 * c) * m] = ycol[row].real();
          Yr[row + static_cast<size_t>(2 * c + 1) * m] = ycol[row].imag();
        }
      }
      const double* ysrc = Yr.data();
      if (Yr.size() <= static_cast<size_t>(m + 1) * (2 * m + 2)) {
        std::memcpy(W.hy.data(), Yr.data(), sizeof(double) * Yr.size());
        ysrc = W.hy.data();
      }
      cuda_check(cudaMemcpyAsync(dQ.p, ysrc, sizeof(double) * Yr.size(), cudaMemcpyHostToDevice, st), "H2D Y");
      std::vector<double> lam(2 * nchk);
      for (int c = 0; c < nchk; ++c) {
        const cplx gam = rz[chk[c]].lambda / vs;  // eigenvalue of the scaled pencil
        cblock[c] = std::abs(gam) > 1.0 ? 1 : 0;  // larger-norm block
        lam[2 * c] = gam.real();
        lam[2 * c + 1] = gam.imag();
      }
      // X = V_m [Re y, Im y] (one DGEMM, row-major) + all residuals in one SpMM pass
      op.ritz_residuals(V, m, dQ.as<double>(), nchk, lam.data(), cblock.data(), dX.as<double>(),
                        dRes.as<double>());
      last_nchk = nchk;
      std::vector<double> rr(2 * nchk);
      cuda_check(cudaMemcpyAsync(rr.data(), dRes.p, sizeof(double) * 2 * nchk, cudaMemcpyDeviceToHost, st),
                 "D2H res");
      cuda_check(cudaStreamSynchronize(st), "sync");
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
    std::vector<int> sel(m, 0);
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
      if (mates_conv && nchk <= m - 1) {
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
        if (p >= keep_target || p + static_cast<int>(g.size()) > m - 1) break;
        for (int i : g) sel[i] = 1;
        p += static_cast<int>(g.size());
      }
      if (p == 0) {  // one cluster fills the whole space: fall back to conjugate pairs
        for (int a = 0; a < m && p < keep_target; ++a) {
          const int i = order[a];
          if (sel[i]) continue;
          int partner = -1;
          double bd = 1e300;
          if (std::abs(rz[i].theta.imag()) > 1e-12 * std::abs(rz[i].theta))
            for (int q = 0; q < m; ++q)
              if (q != i && !sel[q]) {
                const double d = std::abs(rz[q].theta - std::conj(rz[i].theta));
                if (d < bd) bd = d, partner = q;
              }
          if (p + 1 + (partner >= 0) > m - 1) break;
          sel[i] = 1, ++p;
          if (partner >= 0) sel[partner] = 1, ++p;
        }
      }
    }
    // ---- restart: reorder Schur form, real basis of the kept directions ----
    const auto trs0 = now();
    CMat Tr = T, Zr = Z;
    std::vector<int> s2 = sel;
    schur_reorder(Tr, Zr, s2);
    std::vector<double> Qp;
    const int rank = real_basis(Zr, p, Qp);
    if (rank < p) p = rank;
    if (p <= 0) fail(errc::solver, "Krylov-Schur restart lost its basis");
    // T_p = Q_p^T H_m Q_p, b_p = beta_m e_m^T Q_p
    // (column-oriented loops: every inner loop is a contiguous axpy / dot)
    std::vector<double> HQ(static_cast<size_t>(m) * p, 0.0), Tp(static_cast<size_t>(p) * p, 0.0);
    for (int c = 0; c < p; ++c) {
      double* hq = HQ.data() + static_cast<size_t>(c) * m;
      for (int t = 0; t < m; ++t) {
        const double q = Qp[t + static_cast<size_t>(c) * m];
        if (q == 0.0) continue;
        const double* ht = Hm.data() + static_cast<size_t>(t) * m;
        for (int i = 0; i < m; ++i) hq[i] += ht[i] * q;
      }
    }
    for (int c = 0; c < p; ++c) {
      const double* hq = HQ.data() + static_cast<size_t>(c) * m;
      for (int i = 0; i < p; ++i) {
        const double* qi = Qp.data() + static_cast<size_t>(i) * m;
        double s = 0;
        for (int t = 0; t < m; ++t) s += qi[t] * hq[t];
        Tp[i + static_cast<size_t>(c) * p] = s;
      }
    }
    {
      // invariance defect ||H Q_p - Q_p T_p|| / ||H|| (exact restart needs ~eps)
      double dmax = 0, hmax = 0;
      for (double x : Hm) hmax = std::max(hmax, std::fabs(x));
      std::vector<double> rc(m);
      for (int c = 0; c < p; ++c) {
        std::copy(HQ.begin() + static_cast<size_t>(c) * m, HQ.begin() + static_cast<size_t>(c + 1) * m, rc.begin());
        for (int t = 0; t < p; ++t) {
          const double tc = Tp[t + static_cast<size_t>(c) * p];
          const double* qt = Qp.data() + static_cast<size_t>(t) * m;
          for (int i = 0; i < m; ++i) rc[i] -= tc * qt[i];
        }
        for (int i = 0; i < m; ++i) dmax = std::max(dmax, std::fabs(rc[i]));
      }
      res.max_restart_defect = std::max(res.max_restart_defect, dmax / std::max(hmax, 1e-300));
    }
    std::memcpy(W.hq.data(), Qp.data(), sizeof(double) * m * p);
    cuda_check(cudaMemcpyAsync(dQ.p, W.hq.data(), sizeof(double) * m * p, cudaMemcpyHostToDevice, st), "H2D Q");
    op.combine(V, m, dQ.as<double>(), m, p, V2);
    op.combine(BV, m, dQ.as<double>(), m, p, BV2);
    L.n_restart += 1;
    L.macs_restart += static_cast<double>(m) * p * n2;
    std::fill(H.begin(), H.end(), 0.0);
    for (int c = 0; c < p; ++c)
      for (int i = 0; i < p; ++i) Hc(i, c) = Tp[i + static_cast<size_t>(c) * p];
    std::swap(V, V2);
    std::swap(BV, BV2);
    if (deflate) {
      // b = 0 (converged directions deflated); fresh seeded continuation vector
      // (the speculative apply of v_m is discarded)
      pre_applied = false;
      fresh_vector(o.seed + 0x1000003ull * guard_passes, p, V + static_cast<int64_t>(p) * n2,
                   BV + static_cast<int64_t>(p) * n2);
    } else {
      for (int c = 0; c < p; ++c) Hc(p, c) = beta_m * Qp[(m - 1) + static_cast<size_t>(c) * m];
      cuda_check(cudaMemcpyAsync(V + static_cast<int64_t>(p) * n2, V2 + static_cast<int64_t>(m) * n2,
                                 sizeof(double) * n2, cudaMemcpyDeviceToDevice, st), "D2D v");
      cuda_check(cudaMemcpyAsync(BV + static_cast<int64_t>(p) * n2, BV2 + static_cast<int64_t>(m) * n2,
                                 sizeof(double) * n2, cudaMemcpyDeviceToDevice, st), "D2D Bv");
    }
    t_restart += ms_since(trs0);
    if (trace_cycles)
      std::fprintf(stderr, "[eigs] cycle %d: steps %d..%d, checked %d (maybe %d, nconv %d), groups %zu, kept %d%s, "
                   "t ritz %.1f check %.1f restart %.1f sync %.1f ms\n", cycles, k, m, maybe ? nchk : 0, (int)maybe,
                   nconv_now, groups.size(), p, deflate ? " (deflated restart)" : "", t_ritz, t_check, t_restart, t_sync);
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
