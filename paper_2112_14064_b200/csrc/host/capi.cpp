// SPDX-License-Identifier: Apache-2.0
// C-ABI of the B200 build (include/rq_b200.h). Exceptions never cross the
// boundary: every entry point returns an rq::errc value (reference
// types.hpp:14-23) and leaves the message in rq_last_error().
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <array>
#include <future>
#include <mutex>
#include <string>

#include <cuda_runtime_api.h>

#include "../../../include/rq_b200.h"
#include "../engine.hpp"
#include "common.hpp"
#include "io.hpp"
#include "eigs.hpp"
#include "lanczos.hpp"
#include "zeigs.hpp"
#include "dense.hpp"

struct rq_pencil {
  rqb::Pencil P;
  std::unique_ptr<rqb::DevicePencil> dev;  // device-resident K, C, M (P.K/C/M empty)
};
struct rq_mm {
  rqb::CsrFile m;
};
struct rq_symbolic {
  rqb::Symbolic S;
};
struct rq_factor {
  std::unique_ptr<rqb::FactorEngine> owned;
  rqb::FactorEngine* fe = nullptr;
  rqb::DeviceBuffer d_b, d_x;
  int64_t n_complex = -1;  // complex factorization: size of the complex system (the engine holds 2n)
};
struct rq_operator {
  std::unique_ptr<rqb::OperatorEngine> op;
  double norms1[3] = {0, 0, 0};
  rq_factor fac_view;
  rqb::Ledger ledger;  // the last rq_eigs_run
  rqb::Ledger cum;     // every operation on this operator since creation / reset
  rqb::DeviceBuffer d_a, d_b;
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const rqb::Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code());
  } catch (const std::bad_alloc&) {
    g_err = "out of memory";
    return RQ_E_GENERIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RQ_E_GENERIC;
  } catch (...) {
    g_err = "unknown error";
    return RQ_E_GENERIC;
  }
}

void need(const void* p, const char* what) {
  if (!p) rqb::fail(rqb::errc::config, std::string("null argument: ") + what);
}

rqb::VectorSpace space_of(const rq_space_desc* d) {
  need(d, "desc");
  if (d->kind != RQ_SPACE_CURL && d->kind != RQ_SPACE_DIV) rqb::fail(rqb::errc::config, "unknown space kind");
  return rqb::build_space(d->kind == RQ_SPACE_CURL ? rqb::SpaceKind::curl : rqb::SpaceKind::div, d->degree,
                          d->elems, d->levels);
}

// 1-norms (max column sum of |a|) of K, v C and v^2 M in one pass, columns
// accumulated in row order (the sequence norm1 below adds)
std::array<double, 3> norms1_3(int64_t n, const int64_t* rowptr, const int32_t* col, const double* K,
                               const double* C, const double* M, double v) {
  std::vector<double> c0(n, 0.0), c1(n, 0.0), c2(n, 0.0);
  const double vv = v * v;
  for (int64_t r = 0; r < n; ++r)
    for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) {
      const int32_t c = col[k];
      c0[c] += std::fabs(K[k]);
      c1[c] += std::fabs(v * C[k]);
      c2[c] += std::fabs(vv * M[k]);
    }
  std::array<double, 3> out{0.0, 0.0, 0.0};
  for (int64_t j = 0; j < n; ++j) {
    out[0] = std::max(out[0], c0[j]);
    out[1] = std::max(out[1], c1[j]);
    out[2] = std::max(out[2], c2[j]);
  }
  return out;
}

double norm1(int64_t n, const int64_t* rowptr, const int32_t* col, const std::vector<double>& v) {
  std::vector<double> cs(n, 0.0);
  for (int64_t r = 0; r < n; ++r)
    for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) cs[col[k]] += std::fabs(v[k]);
  double m = 0;
  for (double s : cs) m = std::max(m, s);
  return m;
}

}  // namespace

extern "C" {

const char* rq_last_error(void) { return g_err.c_str(); }
const char* rq_version(void) { return "rq_b200 0.1 (sm_100a)"; }

int rq_set_device(int device) {
  return guarded([&] { rqb::cuda_check(cudaSetDevice(device), "cudaSetDevice"); });
}

int rq_pencil_assemble(const rq_space_desc* desc, rq_pencil_t** out) {
  return guarded([&] {
    need(out, "out");
    const rqb::VectorSpace vs = space_of(desc);
    auto p = std::make_unique<rq_pencil>();
    p->P = rqb::assemble_pencil(vs, desc->alpha, desc->beta);
    *out = p.release();
  });
}

int rq_pencil_assemble_acoustic(int degree, int elems, int levels, double rho, double c, double alpha, double beta,
                                int absorbing_edges, rq_pencil_t** out) {
  return guarded([&] {
    need(out, "out");
    const rqb::VectorSpace vs = rqb::build_space(rqb::SpaceKind::div, degree, elems, levels);
    auto p = std::make_unique<rq_pencil>();
    p->P = rqb::assemble_acoustic(vs, rho, c, alpha, beta, absorbing_edges);
    *out = p.release();
  });
}

int rq_pencil_assemble_em(int degree, int elems, int levels, double mu, double eps, int nlayers, const double* layers,
                          double* D_out, rq_pencil_t** out) {
  return guarded([&] {
    need(out, "out");
    if (nlayers < 0 || (nlayers > 0 && !layers)) rqb::fail(rqb::errc::config, "layers");
    std::vector<rqb::EmLayer> L;
    for (int i = 0; i < nlayers; ++i) L.push_back({layers[4 * i], layers[4 * i + 1], layers[4 * i + 2], layers[4 * i + 3]});
    const rqb::VectorSpace vs = rqb::build_space(rqb::SpaceKind::curl, degree, elems, levels);
    auto p = std::make_unique<rq_pencil>();
    std::vector<double> D;
    p->P = rqb::assemble_em(vs, mu, eps, L, &D);
    if (D_out) std::memcpy(D_out, D.data(), sizeof(double) * D.size());
    p->P.C = D;  // the pencil handle carries D in its C slot (C = -i D)
    *out = p.release();
  });
}

int rq_pencil_assemble_device(const rq_space_desc* desc, int resident, rq_pencil_t** out, double* ms) {
  return guarded([&] {
    need(out, "out");
    const rqb::VectorSpace vs = space_of(desc);
    auto p = std::make_unique<rq_pencil>();
    if (resident) p->dev = std::make_unique<rqb::DevicePencil>();
    p->P = rqb::assemble_pencil_device(vs, desc->alpha, desc->beta, ms, p->dev.get());
    *out = p.release();
  });
}

int rq_pencil_dims(const rq_pencil_t* p, int64_t* n_full, int64_t* n_free, int64_t* nnz) {
  return guarded([&] {
    need(p, "pencil");
    if (n_full) *n_full = p->P.n_full;
    if (n_free) *n_free = p->P.n;
    if (nnz) *nnz = p->P.rowptr.back();
  });
}

int rq_pencil_csr(const rq_pencil_t* p, int64_t* rowptr, int32_t* col, double* K, double* C,
                  double* M) {
  return guarded([&] {
    need(p, "pencil");
    const rqb::Pencil& P = p->P;
    if (rowptr) std::memcpy(rowptr, P.rowptr.data(), sizeof(int64_t) * P.rowptr.size());
    if (col) std::memcpy(col, P.col.data(), sizeof(int32_t) * P.col.size());
    if (p->dev) {
      const rqb::DevicePencil& D = *p->dev;
      const size_t b = sizeof(double) * D.nnz;
      int cur = 0;
      rqb::cuda_check(cudaGetDevice(&cur), "cudaGetDevice");
      rqb::cuda_check(cudaSetDevice(D.device), "cudaSetDevice");
      if (K) rqb::cuda_check(cudaMemcpy(K, D.K(), b, cudaMemcpyDeviceToHost), "pencil K D2H");
      if (C) rqb::cuda_check(cudaMemcpy(C, D.C(), b, cudaMemcpyDeviceToHost), "pencil C D2H");
      if (M) rqb::cuda_check(cudaMemcpy(M, D.M(), b, cudaMemcpyDeviceToHost), "pencil M D2H");
      rqb::cuda_check(cudaSetDevice(cur), "cudaSetDevice");
      return;
    }
    if (K) std::memcpy(K, P.K.data(), sizeof(double) * P.K.size());
    if (C) std::memcpy(C, P.C.data(), sizeof(double) * P.C.size());
    if (M) std::memcpy(M, P.M.data(), sizeof(double) * P.M.size());
  });
}

int rq_pencil_supports(const rq_pencil_t* p, int32_t* box, int64_t* free_to_full) {
  return guarded([&] {
    need(p, "pencil");
    if (box) std::memcpy(box, p->P.box.data(), sizeof(int32_t) * p->P.box.size());
    if (free_to_full)
      std::memcpy(free_to_full, p->P.free_to_full.data(), sizeof(int64_t) * p->P.free_to_full.size());
  });
}

void rq_pencil_destroy(rq_pencil_t* p) { delete p; }

int rq_space_dims(const rq_space_desc* desc, int64_t* nx_x, int64_t* ny_x, int64_t* nx_y,
                  int64_t* ny_y) {
  return guarded([&] {
    const rqb::VectorSpace vs = space_of(desc);
    if (nx_x) *nx_x = vs.cx.nx();
    if (ny_x) *ny_x = vs.cx.ny();
    if (nx_y) *nx_y = vs.cy.nx();
    if (ny_y) *ny_y = vs.cy.ny();
  });
}

int rq_space_boundary_mask(const rq_space_desc* desc, int64_t* mask, int64_t* count) {
  return guarded([&] {
    need(count, "count");
    const rqb::VectorSpace vs = space_of(desc);
    const std::vector<int64_t> m = rqb::boundary_mask(vs);
    *count = static_cast<int64_t>(m.size());
    if (mask) std::memcpy(mask, m.data(), sizeof(int64_t) * m.size());
  });
}

int rq_nd_order(int64_t n, const int32_t* box, int elems, int leaf, rq_symbolic_t** out) {
  return guarded([&] {
    need(box, "box");
    need(out, "out");
    auto s = std::make_unique<rq_symbolic>();
    s->S = rqb::nested_dissection(n, box, elems, leaf > 0 ? leaf : 64);
    *out = s.release();
  });
}

int rq_symbolic_stats_get(const rq_symbolic_t* s, rq_symbolic_stats* o) {
  return guarded([&] {
    need(s, "symbolic");
    need(o, "out");
    const rqb::Symbolic& S = s->S;
    o->n = S.n;
    o->nfronts = static_cast<int64_t>(S.fronts.size());
    o->nlevels = static_cast<int64_t>(S.level_fronts.size());
    o->max_front = S.max_front;
    o->max_npiv = S.max_npiv;
    o->nnz_l = S.nnz_l;
    o->nnz_u = S.nnz_u;
    o->pool_doubles = S.pool;
    o->flops_lu = S.flops_lu;
    o->flops_schur = S.flops_schur;
    o->flops_schur_large = S.flops_schur_large;
    o->trisolve_bytes = S.trisolve_bytes;
  });
}

int rq_symbolic_perm(const rq_symbolic_t* s, int32_t* perm) {
  return guarded([&] {
    need(s, "symbolic");
    need(perm, "perm");
    std::memcpy(perm, s->S.perm.data(), sizeof(int32_t) * s->S.perm.size());
  });
}

int rq_symbolic_fronts(const rq_symbolic_t* s, int32_t* parent, int32_t* npiv, int32_t* nf,
                       int32_t* start, int32_t* level) {
  return guarded([&] {
    need(s, "symbolic");
    const auto& F = s->S.fronts;
    for (size_t f = 0; f < F.size(); ++f) {
      if (parent) parent[f] = F[f].parent;
      if (npiv) npiv[f] = F[f].npiv;
      if (nf) nf[f] = F[f].nf;
      if (start) start[f] = F[f].start;
      if (level) level[f] = F[f].level;
    }
  });
}

int rq_symbolic_front_rows(const rq_symbolic_t* s, int64_t f, int32_t* rows) {
  return guarded([&] {
    need(s, "symbolic");
    need(rows, "rows");
    if (f < 0 || f >= static_cast<int64_t>(s->S.fronts.size())) rqb::fail(rqb::errc::dimension, "front id");
    const rqb::Front& F = s->S.fronts[f];
    std::memcpy(rows, s->S.rows.data() + F.rows_off, sizeof(int32_t) * F.nf);
  });
}

void rq_symbolic_destroy(rq_symbolic_t* s) { delete s; }

int rq_factor_create(const rq_symbolic_t* s, int64_t n, const int64_t* rowptr, const int32_t* col,
                     const double* aval, rq_factor_t** out) {
  return guarded([&] {
    need(s, "symbolic");
    need(rowptr, "rowptr");
    need(col, "col");
    need(aval, "aval");
    need(out, "out");
    if (n != s->S.n) rqb::fail(rqb::errc::dimension, "matrix size differs from the symbolic analysis");
    auto f = std::make_unique<rq_factor>();
    f->owned = std::make_unique<rqb::FactorEngine>(s->S, n, rowptr, col, aval);
    f->fe = f->owned.get();
    f->fe->factor();
    *out = f.release();
  });
}

namespace {
// real-equivalent 2n x 2n system of the complex A: unknowns 2k = Re x_k,
// 2k+1 = Im x_k (the cdouble layout), block (i, j) = [[ar, -ai], [ai, ar]]
void complex_equivalent(int64_t n, const int64_t* rowptr, const int32_t* col, const double* are, const double* aim,
                        std::vector<int64_t>& rp2, std::vector<int32_t>& col2, std::vector<double>& v2) {
  const int64_t nnz = rowptr[n];
  if (2 * n > INT32_MAX) rqb::fail(rqb::errc::dimension, "complex system too large for int32 columns");
  rp2.assign(2 * n + 1, 0);
  col2.resize(4 * nnz);
  v2.resize(4 * nnz);
  int64_t q = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int part = 0; part < 2; ++part) {
      rp2[2 * i + part] = q;
      for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
        const int32_t j = col[k];
        const double ar = are[k], ai = aim ? aim[k] : 0.0;
        col2[q] = 2 * j;
        v2[q++] = part == 0 ? ar : ai;
        col2[q] = 2 * j + 1;
        v2[q++] = part == 0 ? -ai : ar;
      }
    }
  rp2[2 * n] = q;
}
}  // namespace

int rq_factor_create_complex(const rq_symbolic_t* s2, int64_t n, const int64_t* rowptr, const int32_t* col,
                             const double* are, const double* aim, rq_factor_t** out) {
  return guarded([&] {
    need(s2, "symbolic");
    need(rowptr, "rowptr");
    need(col, "col");
    need(are, "are");
    need(out, "out");
    if (2 * n != s2->S.n) rqb::fail(rqb::errc::dimension, "the ordering must cover the 2n real-equivalent unknowns");
    std::vector<int64_t> rp2;
    std::vector<int32_t> col2;
    std::vector<double> v2;
    complex_equivalent(n, rowptr, col, are, aim, rp2, col2, v2);
    auto f = std::make_unique<rq_factor>();
    f->owned = std::make_unique<rqb::FactorEngine>(s2->S, 2 * n, rp2.data(), col2.data(), v2.data());
    f->fe = f->owned.get();
    f->n_complex = n;
    f->fe->factor();
    *out = f.release();
  });
}

int rq_factor_refactor_complex(rq_factor_t* f, const double* are, const double* aim, const int64_t* rowptr,
                               const int32_t* col) {
  return guarded([&] {
    need(f, "factor");
    need(are, "are");
    need(rowptr, "rowptr");
    need(col, "col");
    if (f->n_complex < 0) rqb::fail(rqb::errc::config, "not a complex factorization");
    std::vector<int64_t> rp2;
    std::vector<int32_t> col2;
    std::vector<double> v2;
    complex_equivalent(f->n_complex, rowptr, col, are, aim, rp2, col2, v2);
    std::lock_guard<std::mutex> lock(f->fe->mu);
    f->fe->set_values(v2.data());
    f->fe->factor();
  });
}

int rq_factor_refactor(rq_factor_t* f, const double* aval) {
  return guarded([&] {
    need(f, "factor");
    need(aval, "aval");
    if (f->n_complex >= 0) rqb::fail(rqb::errc::config, "complex factorization: use rq_factor_refactor_complex");
    std::lock_guard<std::mutex> lock(f->fe->mu);
    f->fe->factor_streamed(aval);  // the upload overlaps the factorization (chunks in CSR order)
  });
}

int rq_factor_get_info(const rq_factor_t* f, rq_factor_info* o) {
  return guarded([&] {
    need(f, "factor");
    need(o, "out");
    o->swaps = f->fe->last_swaps;
    o->factor_ms = f->fe->last_ms;
    o->gflops = f->fe->last_ms > 0 ? f->fe->sym.flops_lu / (f->fe->last_ms * 1e6) : 0.0;
    o->launches = f->fe->launches_factor;
  });
}

namespace {
int factor_solve_impl(rq_factor_t* f, const double* b, double* x, int nrhs, int block);
}

int rq_factor_solve_ex(rq_factor_t* f, const double* b, double* x, int nrhs, int block) {
  const int rc = guarded([&] {
    need(f, "factor");
    if (f->n_complex >= 0)
      rqb::fail(rqb::errc::config, "complex factorization: use rq_factor_solve_complex (interleaved vectors of n)");
  });
  if (rc != 0) return rc;
  return factor_solve_impl(f, b, x, nrhs, block);
}

namespace {
int factor_solve_impl(rq_factor_t* f, const double* b, double* x, int nrhs, int block) {
  return guarded([&] {
    need(f, "factor");
    need(b, "b");
    need(x, "x");
    if (nrhs < 0) rqb::fail(rqb::errc::dimension, "nrhs must be non-negative");
    if (block < 1 || block > 8) rqb::fail(rqb::errc::config, "block must be 1..8");
    std::lock_guard<std::mutex> lock(f->fe->mu);
    rqb::FactorEngine& fe = *f->fe;
    const int64_t n = fe.n;
    const int w = std::min(block, std::max(nrhs, 1));
    if (f->d_b.bytes < sizeof(double) * n * w) f->d_b.alloc(sizeof(double) * n * w);
    if (f->d_x.bytes < sizeof(double) * n * w) f->d_x.alloc(sizeof(double) * n * w);
    for (int r = 0; r < nrhs; r += w) {
      const int k = std::min(w, nrhs - r);
      rqb::cuda_check(cudaMemcpyAsync(f->d_b.p, b + static_cast<int64_t>(r) * n, sizeof(double) * n * k,
                                      cudaMemcpyHostToDevice, fe.stream), "H2D b");
      if (block == 1)
        fe.solve_device(f->d_b.as<double>(), f->d_x.as<double>(), 1.0);
      else
        rqb::rqb_msolve_enqueue(fe, f->d_b.as<double>(), n, k, f->d_x.as<double>(), n, 1.0, nullptr, 0, 0.0,
                                nullptr);
      rqb::cuda_check(cudaMemcpyAsync(x + static_cast<int64_t>(r) * n, f->d_x.p, sizeof(double) * n * k,
                                      cudaMemcpyDeviceToHost, fe.stream), "D2H x");
    }
    rqb::cuda_check(cudaStreamSynchronize(fe.stream), "solve sync");
    fe.check_sweeps();
    rqb::rqb_msolve_check(fe);
  });
}

}  // namespace

int rq_factor_solve_complex(rq_factor_t* f, const double* b, double* x, int nrhs) {
  const int rc = guarded([&] {
    need(f, "factor");
    if (f->n_complex < 0) rqb::fail(rqb::errc::config, "not a complex factorization");
  });
  if (rc != 0) return rc;
  // interleaved {re, im} vectors are exactly the real-equivalent unknowns
  return factor_solve_impl(f, b, x, nrhs, nrhs > 1 ? 8 : 1);
}

int rq_factor_solve(rq_factor_t* f, const double* b, double* x, int nrhs) {
  return rq_factor_solve_ex(f, b, x, nrhs, nrhs > 1 ? 8 : 1);
}

int rq_factor_front_export(const rq_factor_t* f, int64_t front, double* dense, int32_t* ipiv,
                           int64_t* ld_out) {
  return guarded([&] {
    need(f, "factor");
    const rqb::FactorEngine& fe = *f->fe;
    if (front < 0 || front >= static_cast<int64_t>(fe.fronts_h.size()))
      rqb::fail(rqb::errc::dimension, "front id");
    const rqb::FrontDev& F = fe.fronts_h[front];
    if (ld_out) *ld_out = F.ld;
    if (dense)
      rqb::cuda_check(cudaMemcpy(dense, fe.d_pool.as<double>() + F.off, sizeof(double) * F.ld * F.nf,
                                 cudaMemcpyDeviceToHost), "D2H front");
    if (ipiv && F.npiv > 0) {
      rqb::cuda_check(cudaMemcpy(ipiv, fe.d_ipiv.as<int32_t>() + F.start, sizeof(int32_t) * F.npiv,
                                 cudaMemcpyDeviceToHost), "D2H ipiv");
    }
  });
}

int rq_factor_profile(rq_factor_t* f, double* ms, int64_t* launches, double* work) {
  return guarded([&] {
    need(f, "factor");
    need(ms, "ms");
    need(launches, "launches");
    need(work, "work");
    std::lock_guard<std::mutex> lock(f->fe->mu);
    f->fe->profile(ms, launches, work);
  });
}

int rq_factor_dag_profile(rq_factor_t* f, double* out) {
  return guarded([&] {
    need(f, "factor");
    need(out, "out");
    std::lock_guard<std::mutex> lock(f->fe->mu);
    rqb::rqb_dag_profile(*f->fe, out);
  });
}

int rq_factor_bench_updcb(rq_factor_t* f, int front, int reps, double* out) {
  return guarded([&] {
    need(f, "factor");
    need(out, "out");
    std::lock_guard<std::mutex> lock(f->fe->mu);
    rqb::rqb_dag_bench_updcb(*f->fe, front, reps, out);
  });
}

void rq_factor_destroy(rq_factor_t* f) { delete f; }

namespace {
void finish_operator(rq_operator* o) {
  rqb::charge_factor(o->cum, *o->op);  // build_operator: N_fa = 1
  o->fac_view.fe = o->op->fac.get();
  o->d_a.alloc(sizeof(double) * 2 * o->op->n);
  o->d_b.alloc(sizeof(double) * 2 * o->op->n);
}
}  // namespace

int rq_operator_create(int64_t n, const int64_t* rowptr, const int32_t* col, const double* K,
                       const double* C, const double* M, const rq_symbolic_t* s,
                       const rq_operator_opts* opts, rq_operator_t** out) {
  return guarded([&] {
    need(rowptr, "rowptr");
    need(col, "col");
    need(K, "K");
    need(C, "C");
    need(M, "M");
    need(s, "symbolic");
    need(opts, "opts");
    need(out, "out");
    if (!std::isfinite(opts->sigma)) rqb::fail(rqb::errc::config, "shift must be finite and real");
    auto o = std::make_unique<rq_operator>();
    // the residual 1-norms of K, varsigma C, varsigma^2 M (true column sums: the
    // host pencil need not be symmetric) on a host thread while the engine
    // uploads the pencil and factors Q(s)
    const bool scaling = opts->scaling != 0;
    auto norms = std::async(std::launch::async, [&] {
      double v = 1.0;
      if (scaling) {
        double mk = 0, mm = 0;
        for (int64_t k = 0; k < rowptr[n]; ++k) mk = std::max(mk, std::fabs(K[k])), mm = std::max(mm, std::fabs(M[k]));
        if (mm > 0) v = std::sqrt(mk / mm);
      }
      return norms1_3(n, rowptr, col, K, C, M, v);
    });
    try {
      o->op = std::make_unique<rqb::OperatorEngine>(n, rowptr, col, K, C, M, s->S, opts->sigma, scaling);
    } catch (...) {
      norms.wait();
      throw;
    }
    const std::array<double, 3> nr = norms.get();
    for (int i = 0; i < 3; ++i) o->norms1[i] = nr[i];
    finish_operator(o.get());
    *out = o.release();
  });
}

int rq_operator_create_pencil(const rq_pencil_t* p, const rq_symbolic_t* s,
                              const rq_operator_opts* opts, rq_operator_t** out) {
  if (p && !p->dev)
    return rq_operator_create(p->P.n, p->P.rowptr.data(), p->P.col.data(), p->P.K.data(),
                              p->P.C.data(), p->P.M.data(), s, opts, out);
  return guarded([&] {
    need(p, "pencil");
    need(s, "symbolic");
    need(opts, "opts");
    need(out, "out");
    if (!std::isfinite(opts->sigma)) rqb::fail(rqb::errc::config, "shift must be finite and real");
    auto o = std::make_unique<rq_operator>();
    o->op = std::make_unique<rqb::OperatorEngine>(*p->dev, p->P.rowptr.data(), p->P.col.data(), s->S,
                                                  opts->sigma, opts->scaling != 0, o->norms1);
    finish_operator(o.get());
    *out = o.release();
  });
}

double rq_operator_varsigma(const rq_operator_t* op) { return op ? op->op->varsigma : 0.0; }

rq_factor_t* rq_operator_factor(rq_operator_t* op) { return op ? &op->fac_view : nullptr; }

void rq_operator_destroy(rq_operator_t* op) { delete op; }

int rq_operator_time(rq_operator_t* o, int what, int iters, int param, double* ms_per_call) {
  return guarded([&] {
    need(o, "op");
    need(ms_per_call, "ms");
    std::lock_guard<std::mutex> lock(o->op->fac->mu);
    if (iters < 1) rqb::fail(rqb::errc::config, "iters must be positive");
    *ms_per_call = o->op->time_op(what, iters, param);
  });
}

int rq_operator_apply(rq_operator_t* o, const double* v, double* r) {
  return guarded([&] {
    need(o, "op");
    need(v, "v");
    need(r, "r");
    std::lock_guard<std::mutex> lock(o->op->fac->mu);
    rqb::OperatorEngine& op = *o->op;
    const int64_t n2 = 2 * op.n;
    rqb::cuda_check(cudaMemcpyAsync(o->d_a.p, v, sizeof(double) * n2, cudaMemcpyHostToDevice, op.stream), "H2D");
    op.apply(o->d_a.as<double>(), o->d_b.as<double>());
    rqb::cuda_check(cudaMemcpyAsync(r, o->d_b.p, sizeof(double) * n2, cudaMemcpyDeviceToHost, op.stream), "D2H");
    rqb::cuda_check(cudaStreamSynchronize(op.stream), "sync");
    op.fac->check_sweeps();
    rqb::charge_apply(o->cum, op);
  });
}

int rq_operator_b_inner(rq_operator_t* o, const double* x, const double* y, double* out) {
  return guarded([&] {
    need(o, "op");
    need(x, "x");
    need(y, "y");
    need(out, "out");
    std::lock_guard<std::mutex> lock(o->op->fac->mu);
    rqb::OperatorEngine& op = *o->op;
    const int64_t n2 = 2 * op.n;
    rqb::DeviceBuffer dw, ds;
    dw.alloc(sizeof(double) * n2);
    ds.alloc(sizeof(double));
    rqb::cuda_check(cudaMemcpyAsync(o->d_a.p, x, sizeof(double) * n2, cudaMemcpyHostToDevice, op.stream), "H2D");
    rqb::cuda_check(cudaMemcpyAsync(o->d_b.p, y, sizeof(double) * n2, cudaMemcpyHostToDevice, op.stream), "H2D");
    op.bvec(o->d_b.as<double>(), dw.as<double>());
    op.dot2n(o->d_a.as<double>(), dw.as<double>(), ds.as<double>());
    rqb::cuda_check(cudaMemcpyAsync(out, ds.p, sizeof(double), cudaMemcpyDeviceToHost, op.stream), "D2H");
    rqb::cuda_check(cudaStreamSynchronize(op.stream), "sync");
    rqb::charge_bproduct(o->cum, op);  // b_inner
    rqb::charge_vv2n(o->cum, op, 1);
  });
}

int rq_operator_spmv(rq_operator_t* o, int which, const double* x, double* y) {
  return guarded([&] {
    need(o, "op");
    need(x, "x");
    need(y, "y");
    std::lock_guard<std::mutex> lock(o->op->fac->mu);
    if (which < 0 || which > 3) rqb::fail(rqb::errc::config, "which must be 0..3");
    rqb::OperatorEngine& op = *o->op;
    const int64_t n = op.n;
    rqb::cuda_check(cudaMemcpyAsync(o->d_a.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, op.stream), "H2D");
    op.spmv(which, o->d_a.as<double>(), o->d_b.as<double>());
    rqb::cuda_check(cudaMemcpyAsync(y, o->d_b.p, sizeof(double) * n, cudaMemcpyDeviceToHost, op.stream), "D2H");
    rqb::cuda_check(cudaStreamSynchronize(op.stream), "sync");
    rqb::charge_bproduct(o->cum, op);  // rq::spmv: one mv of nnz MACs (sparse.cpp:59-62)
  });
}

int rq_operator_arnoldi(rq_operator_t* o, const double* v1, int m, double* V, double* H) {
  return guarded([&] {
    need(o, "op");
    need(v1, "v1");
    std::lock_guard<std::mutex> lock(o->op->fac->mu);
    if (m < 1 || m > 512) rqb::fail(rqb::errc::config, "m must be in [1, 512]");
    rqb::OperatorEngine& op = *o->op;
    const int64_t n2 = 2 * op.n;
    rqb::DeviceBuffer dV, dr, dw, dh, dbeta;
    dV.alloc(sizeof(double) * (m + 1) * n2);
    dr.alloc(sizeof(double) * n2);
    dw.alloc(sizeof(double) * n2);
    dh.alloc(sizeof(double) * 2 * (m + 1) * m);
    dbeta.alloc(sizeof(double) * (m + 1));
    double* dVp = dV.as<double>();
    rqb::cuda_check(cudaMemcpyAsync(dr.p, v1, sizeof(double) * n2, cudaMemcpyHostToDevice, op.stream), "H2D");
    op.bvec(dr.as<double>(), dw.as<double>());
    op.bnorm_normalize(dr.as<double>(), dw.as<double>(), dbeta.as<double>() + m, dVp);
    for (int j = 0; j < m; ++j) {
      double* hA = dh.as<double>() + static_cast<int64_t>(j) * (m + 1);
      double* hB = hA + static_cast<int64_t>(m) * (m + 1);
      op.apply(dVp + j * n2, dr.as<double>());
      for (int pass = 0; pass < 2; ++pass) {
        double* h = pass ? hB : hA;
        op.bvec(dr.as<double>(), dw.as<double>());
        op.gemv_t(dVp, j + 1, dw.as<double>(), h);
        op.gemv_n(dVp, j + 1, h, dr.as<double>(), nullptr);
      }
      op.bvec(dr.as<double>(), dw.as<double>());
      op.bnorm_normalize(dr.as<double>(), dw.as<double>(), dbeta.as<double>() + j, dVp + (j + 1) * n2);
    }
    std::vector<double> hh(2 * (m + 1) * m), beta(m + 1);
    rqb::cuda_check(cudaMemcpyAsync(hh.data(), dh.p, sizeof(double) * hh.size(), cudaMemcpyDeviceToHost, op.stream), "D2H");
    rqb::cuda_check(cudaMemcpyAsync(beta.data(), dbeta.p, sizeof(double) * beta.size(), cudaMemcpyDeviceToHost, op.stream), "D2H");
    if (V)
      rqb::cuda_check(cudaMemcpyAsync(V, dV.p, sizeof(double) * (m + 1) * n2, cudaMemcpyDeviceToHost, op.stream), "D2H");
    rqb::cuda_check(cudaStreamSynchronize(op.stream), "sync");
    // arnoldi_run: v1 B-normalised, then m steps
    rqb::charge_bproduct(o->cum, op);
    rqb::charge_vv2n(o->cum, op, 1);
    for (int j = 0; j < m; ++j) {
      rqb::charge_apply(o->cum, op);
      for (int pass = 0; pass < 3; ++pass) rqb::charge_bproduct(o->cum, op);
      rqb::charge_vv2n(o->cum, op, 4 * (j + 1) + 1);
    }
    if (H) {
      std::fill(H, H + (m + 1) * m, 0.0);
      for (int j = 0; j < m; ++j) {
        for (int i = 0; i <= j; ++i)
          H[i + j * (m + 1)] = hh[i + j * (m + 1)] + hh[static_cast<size_t>(m) * (m + 1) + i + j * (m + 1)];
        H[j + 1 + j * (m + 1)] = beta[j];
      }
    }
  });
}

int rq_eigs_run(rq_operator_t* o, const rq_eigs_opts* opts, double* lam_re, double* lam_im,
                double* resid, double* vec_re, double* vec_im, rq_eigs_info* info) {
  int nconv_out = 0;
  bool partial = false;
  const int rc = guarded([&] {
    need(o, "op");
    need(opts, "opts");
    std::lock_guard<std::mutex> lock(o->op->fac->mu);
    rqb::EigsOptions eo;
    eo.nev = opts->nev;
    eo.m = opts->m;
    eo.tol = opts->tol;
    eo.seed = opts->seed;
    eo.max_restarts = opts->max_restarts > 0 ? opts->max_restarts : 100;
    eo.guard = opts->guard;
    if (const char* e = std::getenv("RQB_GUARD_CLUSTER")) eo.guard_single_cluster = std::atoi(e);
    eo.profile = opts->profile;
    eo.block = opts->block;
    if (const char* e = std::getenv("RQB_RQ_REFINE")) eo.refine = std::atoi(e);
    eo.want_vectors = (vec_re && vec_im) ? 1 : 0;
    o->ledger = rqb::Ledger{};
    rqb::EigsResult r = rqb::solve_quadratic_device(*o->op, eo, o->ledger, o->norms1);
    o->cum.add(o->ledger, false);  // the factorization was charged when the operator was built
    const int nout = static_cast<int>(r.lambda.size());
    for (int i = 0; i < nout && i < opts->nev; ++i) {
      if (lam_re) lam_re[i] = r.lambda[i].real();
      if (lam_im) lam_im[i] = r.lambda[i].imag();
      if (resid) resid[i] = r.resid[i];
    }
    if (eo.want_vectors && !r.vec_re.empty()) {
      std::memcpy(vec_re, r.vec_re.data(), sizeof(double) * r.vec_re.size());
      std::memcpy(vec_im, r.vec_im.data(), sizeof(double) * r.vec_im.size());
    }
    nconv_out = r.nconv;
    if (info) {
      rq_eigs_info& I = *info;
      I.nconv = r.nconv;
      I.restarts = r.cycles;
      I.guard_passes = r.guard_passes;
      const rqb::Ledger& L = o->ledger;
      I.n_fa = L.n_fa;
      I.n_fb = L.n_fb;
      I.n_mv = L.n_mv;
      I.n_vv = L.n_vv;
      I.n_check = L.n_check;
      I.n_restart = L.n_restart;
      I.macs_fa = L.macs_fa;
      I.macs_fb = L.macs_fb;
      I.macs_mv = L.macs_mv;
      I.macs_vv = L.macs_vv;
      I.macs_check = L.macs_check;
      I.macs_restart = L.macs_restart;
      I.t_total_ms = r.t_total_ms;
      I.t_factor_ms = o->op->fac->last_ms;
      I.t_solve_ms = r.t_solve_ms;
      I.t_spmv_ms = 0;
      I.t_orth_ms = r.t_orth_ms;
      I.t_host_ms = 0;
      I.launches = r.launches;
      I.restart_defect = r.max_restart_defect;
      I.t_ritz_ms = r.t_ritz_ms;
      I.t_check_ms = r.t_check_ms;
      I.t_restart_ms = r.t_restart_ms;
      I.t_sync_ms = r.t_sync_ms;
    }
    partial = r.nconv < opts->nev;
  });
  if (rc != 0) return rc;
  if (partial) {
    g_err = "solve_quadratic: only " + std::to_string(nconv_out) + " pairs converged within max_restarts";
    return RQ_E_SOLVER;
  }
  return 0;
}

int rq_operator_release_workspace(rq_operator_t* o) {
  return guarded([&] {
    need(o, "op");
    std::lock_guard<std::mutex> lock(o->op->fac->mu);
    rqb::cuda_check(cudaStreamSynchronize(o->op->stream), "sync");
    o->op->eig_ws.reset();
  });
}

int rq_operator_ledger(const rq_operator_t* o, double* out) {
  return guarded([&] {
    need(o, "op");
    need(out, "out");
    std::lock_guard<std::mutex> lock(o->op->fac->mu);
    o->cum.get(out);
  });
}

int rq_operator_ledger_json(const rq_operator_t* o, char* buf, size_t len) {
  return guarded([&] {
    need(o, "op");
    need(buf, "buf");
    const std::string s = o->cum.to_json();
    if (s.size() + 1 > len) rqb::fail(rqb::errc::dimension, "ledger buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int rq_operator_ledger_reset(rq_operator_t* o) {
  return guarded([&] {
    need(o, "op");
    o->cum = rqb::Ledger{};
  });
}

int rq_eigs_ledger_json(const rq_operator_t* o, char* buf, size_t len) {
  return guarded([&] {
    need(o, "op");
    need(buf, "buf");
    const std::string s = o->ledger.to_json();
    if (s.size() + 1 > len) rqb::fail(rqb::errc::dimension, "buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

// ---------------------------------------------------------------------------
// scale_pencil, ritz_extract, krylov_schur_restart

int rq_scale_pencil(int64_t nnz, const double* K, const double* C, const double* M, double* varsigma,
                    double* Cs, double* Ms) {
  return guarded([&] {
    need(K, "K");
    need(C, "C");
    need(M, "M");
    need(varsigma, "varsigma");
    double mk = 0, mm = 0;
    for (int64_t k = 0; k < nnz; ++k) mk = std::max(mk, std::fabs(K[k])), mm = std::max(mm, std::fabs(M[k]));
    if (!(mm > 0)) rqb::fail(rqb::errc::domain, "scale_pencil: zero M norm");
    const double v = std::sqrt(mk / mm), v2 = v * v;  // the rule OperatorEngine applies (krylov.cu)
    *varsigma = v;
    if (Cs)
      for (int64_t k = 0; k < nnz; ++k) Cs[k] = v * C[k];
    if (Ms)
      for (int64_t k = 0; k < nnz; ++k) Ms[k] = v2 * M[k];
  });
}

namespace {

// wanted order: nearest the shift first (|lambda - sigma|), conjugate pairs
// adjacent with the positive imaginary part first (the order solve_quadratic
// uses, eigs.cpp)
std::vector<int> wanted_order(const std::vector<rqb::cplx>& lam, double sigma) {
  std::vector<int> order(lam.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    const double da = std::abs(lam[a] - sigma), db = std::abs(lam[b] - sigma);
    if (da != db) return da < db;
    return lam[a].imag() > lam[b].imag();
  });
  return order;
}

struct RitzData {
  rqb::CMat T, Z, Y;
  std::vector<rqb::cplx> theta, lam;
  std::vector<int> order;
  std::vector<double> Hm;
  double beta = 0;
};

RitzData ritz(const double* H, int m, double sigma, double varsigma) {
  RitzData R;
  R.Hm.resize(static_cast<size_t>(m) * m);
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < m; ++i) R.Hm[i + static_cast<size_t>(j) * m] = H[i + static_cast<size_t>(j) * (m + 1)];
  R.beta = H[m + static_cast<size_t>(m - 1) * (m + 1)];
  if (!rqb::complex_schur(R.Hm, m, R.T, R.Z)) rqb::fail(rqb::errc::solver, "Hessenberg QR did not converge");
  R.Y = rqb::triangular_eigvecs(R.T);
  R.theta.resize(m);
  R.lam.resize(m);
  for (int i = 0; i < m; ++i) {
    R.theta[i] = R.T(i, i);
    R.lam[i] = sigma + varsigma / R.theta[i];  // lambda = varsigma (sigma / varsigma + 1 / theta)
  }
  R.order = wanted_order(R.lam, sigma);
  return R;
}

}  // namespace

int rq_ritz_extract(const double* H, int m, double sigma, double varsigma, double* theta, double* lam, double* est,
                    double* Y) {
  return guarded([&] {
    need(H, "H");
    if (m < 1 || m > 512) rqb::fail(rqb::errc::config, "m must be in [1, 512]");
    if (!(varsigma > 0)) rqb::fail(rqb::errc::config, "varsigma must be positive");
    const RitzData R = ritz(H, m, sigma, varsigma);
    for (int a = 0; a < m; ++a) {
      const int i = R.order[a];
      // y = Z Y[:, i] (Y upper triangular), unit 2-norm
      std::vector<rqb::cplx> y(m, 0.0);
      for (int t = 0; t <= i; ++t)
        for (int row = 0; row < m; ++row) y[row] += R.Z(row, t) * R.Y(t, i);
      if (theta) theta[2 * a] = R.theta[i].real(), theta[2 * a + 1] = R.theta[i].imag();
      if (lam) lam[2 * a] = R.lam[i].real(), lam[2 * a + 1] = R.lam[i].imag();
      if (est) est[a] = std::abs(R.beta * y[m - 1]);
      if (Y)
        for (int row = 0; row < m; ++row) {
          Y[2 * (row + static_cast<size_t>(a) * m)] = y[row].real();
          Y[2 * (row + static_cast<size_t>(a) * m) + 1] = y[row].imag();
        }
    }
  });
}

int rq_operator_krylov_schur_restart(rq_operator_t* o, int m, int keep, double* V, double* H, int* p_out) {
  return guarded([&] {
    need(o, "op");
    need(V, "V");
    need(H, "H");
    need(p_out, "p_out");
    std::lock_guard<std::mutex> lock(o->op->fac->mu);
    rqb::OperatorEngine& op = *o->op;
    if (m < 2 || m > 512 || m >= 2 * op.n) rqb::fail(rqb::errc::config, "m must be in [2, min(512, 2n - 1)]");
    if (keep < 1) rqb::fail(rqb::errc::config, "keep must be positive");
    if (keep >= m) {  // identity restart
      *p_out = m;
      return;
    }
    const int64_t n2 = 2 * op.n;
    const RitzData R = ritz(H, m, op.sigma * op.varsigma, op.varsigma);
    // the `keep` wanted directions, closed under conjugation
    std::vector<int> sel(m, 0);
    int p = 0;
    for (int a = 0; a < m && p < keep; ++a) {
      const int i = R.order[a];
      if (sel[i]) continue;
      int partner = -1;
      if (std::abs(R.theta[i].imag()) > 1e-12 * std::abs(R.theta[i])) {
        double bd = 1e300;
        for (int q = 0; q < m; ++q)
          if (q != i && !sel[q] && std::abs(R.theta[q] - std::conj(R.theta[i])) < bd)
            bd = std::abs(R.theta[q] - std::conj(R.theta[i])), partner = q;
      }
      if (p + 1 + (partner >= 0) > m - 1) break;
      sel[i] = 1, ++p;
      if (partner >= 0) sel[partner] = 1, ++p;
    }
    if (p == 0) rqb::fail(rqb::errc::solver, "krylov_schur_restart: nothing to keep");
    rqb::CMat Tr = R.T, Zr = R.Z;
    rqb::schur_reorder(Tr, Zr, sel);
    std::vector<double> Qp;
    p = rqb::real_basis(Zr, p, Qp);
    if (p <= 0) rqb::fail(rqb::errc::solver, "krylov_schur_restart lost its basis");
    // T_p = Q_p^T H_m Q_p, b_p = beta e_m^T Q_p
    std::vector<double> Tp(static_cast<size_t>(p) * p, 0.0), HQ(static_cast<size_t>(m) * p, 0.0);
    for (int c = 0; c < p; ++c)
      for (int t = 0; t < m; ++t) {
        const double q = Qp[t + static_cast<size_t>(c) * m];
        for (int i = 0; i < m; ++i) HQ[i + static_cast<size_t>(c) * m] += R.Hm[i + static_cast<size_t>(t) * m] * q;
      }
    for (int c = 0; c < p; ++c)
      for (int i = 0; i < p; ++i) {
        double s = 0;
        for (int t = 0; t < m; ++t) s += Qp[t + static_cast<size_t>(i) * m] * HQ[t + static_cast<size_t>(c) * m];
        Tp[i + static_cast<size_t>(c) * p] = s;
      }
    // V_p = V_m Q_p on the device (vq_gemm); v_{p+1} = v_{m+1}
    rqb::DeviceBuffer dV, dQ, dX;
    dV.alloc(sizeof(double) * (m + 1) * n2);
    dQ.alloc(sizeof(double) * m * p);
    dX.alloc(sizeof(double) * p * n2);
    rqb::cuda_check(cudaMemcpyAsync(dV.p, V, sizeof(double) * (m + 1) * n2, cudaMemcpyHostToDevice, op.stream), "H2D V");
    rqb::cuda_check(cudaMemcpyAsync(dQ.p, Qp.data(), sizeof(double) * m * p, cudaMemcpyHostToDevice, op.stream), "H2D Q");
    op.combine(dV.as<double>(), m, dQ.as<double>(), m, p, dX.as<double>());
    rqb::cuda_check(cudaMemcpyAsync(V + static_cast<int64_t>(p) * n2, dV.as<double>() + static_cast<int64_t>(m) * n2,
                                    sizeof(double) * n2, cudaMemcpyDeviceToHost, op.stream), "D2H v");
    rqb::cuda_check(cudaMemcpyAsync(V, dX.p, sizeof(double) * p * n2, cudaMemcpyDeviceToHost, op.stream), "D2H V");
    rqb::cuda_check(cudaStreamSynchronize(op.stream), "sync");
    std::fill(H, H + static_cast<size_t>(m + 1) * m, 0.0);
    for (int c = 0; c < p; ++c) {
      for (int i = 0; i < p; ++i) H[i + static_cast<size_t>(c) * (m + 1)] = Tp[i + static_cast<size_t>(c) * p];
      H[p + static_cast<size_t>(c) * (m + 1)] = R.beta * Qp[(m - 1) + static_cast<size_t>(c) * m];
    }
    *p_out = p;
    o->cum.n_restart += 1;
    o->cum.macs_restart += static_cast<double>(m) * p * n2;
  });
}


int rq_mm_write(int64_t n, const int64_t* rowptr, const int32_t* col, const double* re, const double* im,
                const char* path) {
  return guarded([&] {
    need(rowptr, "rowptr");
    need(path, "path");
    if (n < 0) rqb::fail(rqb::errc::dimension, "negative dimension");
    if (rowptr[n] > 0) {
      need(col, "col");
      need(re, "re");
    }
    rqb::write_mm_csr(n, rowptr, col, re, im, path);
  });
}

int rq_mm_write_vector(int64_t n, const double* re, const double* im, const char* path) {
  return guarded([&] {
    need(path, "path");
    if (n < 0) rqb::fail(rqb::errc::dimension, "negative dimension");
    if (n > 0) need(re, "re");
    rqb::write_mm_vector(n, re, im, path);
  });
}

int rq_mm_read(const char* path, rq_mm_t** out) {
  return guarded([&] {
    need(path, "path");
    need(out, "out");
    auto m = std::make_unique<rq_mm>();
    m->m = rqb::read_mm_csr(path);
    *out = m.release();
  });
}

int rq_mm_dims(const rq_mm_t* m, int64_t* n, int64_t* nnz, int* complex_values) {
  return guarded([&] {
    need(m, "mm");
    if (n) *n = m->m.n;
    if (nnz) *nnz = static_cast<int64_t>(m->m.col.size());
    if (complex_values) *complex_values = m->m.complex_values ? 1 : 0;
  });
}

int rq_mm_csr(const rq_mm_t* m, int64_t* rowptr, int32_t* col, double* re, double* im) {
  return guarded([&] {
    need(m, "mm");
    const rqb::CsrFile& c = m->m;
    if (rowptr) std::memcpy(rowptr, c.rowptr.data(), sizeof(int64_t) * c.rowptr.size());
    if (col) std::memcpy(col, c.col.data(), sizeof(int32_t) * c.col.size());
    if (re) std::memcpy(re, c.re.data(), sizeof(double) * c.re.size());
    if (im) std::memcpy(im, c.im.data(), sizeof(double) * c.im.size());
  });
}

void rq_mm_destroy(rq_mm_t* m) { delete m; }

int rq_pencil_write_mm(const rq_pencil_t* p, const char* prefix) {
  return guarded([&] {
    need(p, "pencil");
    need(prefix, "prefix");
    const rqb::Pencil& P = p->P;
    const int64_t nnz = P.rowptr.back();
    std::vector<double> vals[3];
    const double* src[3] = {P.K.data(), P.C.data(), P.M.data()};
    if (p->dev) {  // device-resident values: one copy out
      int cur = 0;
      rqb::cuda_check(cudaGetDevice(&cur), "cudaGetDevice");
      rqb::cuda_check(cudaSetDevice(p->dev->device), "cudaSetDevice");
      const double* d[3] = {p->dev->K(), p->dev->C(), p->dev->M()};
      for (int w = 0; w < 3; ++w) {
        vals[w].resize(nnz);
        rqb::cuda_check(cudaMemcpy(vals[w].data(), d[w], sizeof(double) * nnz, cudaMemcpyDeviceToHost), "D2H");
        src[w] = vals[w].data();
      }
      rqb::cuda_check(cudaSetDevice(cur), "cudaSetDevice");
    }
    const char* names[3] = {"K.mtx", "C.mtx", "M.mtx"};
    for (int w = 0; w < 3; ++w)
      rqb::write_mm_csr(P.n, P.rowptr.data(), P.col.data(), src[w], nullptr, std::string(prefix) + names[w]);
  });
}

int rq_eigenpairs_json(int n, const double* re, const double* im, const double* residual, char* buf,
                       int64_t cap, int64_t* len) {
  return guarded([&] {
    if (n < 0) rqb::fail(rqb::errc::dimension, "negative count");
    if (n > 0) {
      need(re, "re");
      need(im, "im");
      need(residual, "residual");
    }
    const std::string s = rqb::eigenpairs_json(n, re, im, residual);
    if (len) *len = static_cast<int64_t>(s.size());
    if (buf) {
      if (cap < static_cast<int64_t>(s.size()) + 1) rqb::fail(rqb::errc::dimension, "buffer too small");
      std::memcpy(buf, s.c_str(), s.size() + 1);
    }
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// solve_generalized_hermitian
struct rq_gh {
  std::unique_ptr<rqb::GhEngine> E;
  double normA1 = 0.0, normB1 = 0.0;
};

int rq_gh_create(int64_t n, const int64_t* rowptr, const int32_t* col, const double* A, const double* B,
                 const rq_symbolic_t* s, double shift, rq_gh_t** out) {
  return guarded([&] {
    need(rowptr, "rowptr");
    need(col, "col");
    need(A, "A");
    need(B, "B");
    need(s, "symbolic");
    need(out, "out");
    if (!std::isfinite(shift)) rqb::fail(rqb::errc::config, "shift must be finite and real");
    if (s->S.n != n) rqb::fail(rqb::errc::dimension, "symbolic / matrix dimension mismatch");
    auto h = std::make_unique<rq_gh>();
    h->E = std::make_unique<rqb::GhEngine>(n, rowptr, col, A, B, s->S, shift);
    const int64_t nnz = rowptr[n];
    h->normA1 = norm1(n, rowptr, col, std::vector<double>(A, A + nnz));
    h->normB1 = norm1(n, rowptr, col, std::vector<double>(B, B + nnz));
    *out = h.release();
  });
}

int rq_gh_run(rq_gh_t* h, const rq_gh_opts* opts, double* lam, double* resid, double* vec, rq_gh_info* info) {
  return guarded([&] {
    need(h, "handle");
    need(opts, "opts");
    need(lam, "lam");
    need(resid, "resid");
    std::lock_guard<std::mutex> lock(h->E->fac->mu);
    rqb::GhOptions o;
    o.nev = opts->nev;
    o.m = opts->m;
    o.tol = opts->tol;
    o.seed = opts->seed;
    o.max_restarts = opts->max_restarts > 0 ? opts->max_restarts : 100;
    o.want_vectors = vec ? 1 : 0;
    const auto t0 = std::chrono::steady_clock::now();
    const rqb::GhResult r = rqb::solve_generalized_hermitian_device(*h->E, o, h->normA1, h->normB1);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    const int nout = std::min(o.nev, static_cast<int>(r.lam.size()));
    for (int i = 0; i < o.nev; ++i) {
      lam[i] = i < nout ? r.lam[i] : 0.0;
      resid[i] = i < nout ? r.resid[i] : 1.0;
    }
    if (vec && !r.vec.empty()) std::memcpy(vec, r.vec.data(), sizeof(double) * h->E->n * nout);
    if (info) {
      info->nconv = r.nconv;
      info->cycles = r.cycles;
      info->restarts = r.restarts;
      info->lanczos_defect = r.lanczos_defect;
      info->sym_defect = r.sym_defect;
      info->launches = r.launches;
      info->t_total_ms = ms;
    }
    if (!r.converged)
      rqb::fail(rqb::errc::solver, "solve_generalized_hermitian: only " + std::to_string(r.nconv) +
                                       " pairs converged within max_restarts");
  });
}

void rq_gh_destroy(rq_gh_t* h) { delete h; }

// ---------------------------------------------------------------------------
// complex pencils / complex shifts
struct rq_zeig {
  std::unique_ptr<rqb::ZOperatorEngine> E;
  double norms1[3] = {0, 0, 0};
};

int rq_zeig_create(const rq_symbolic_t* s2, int64_t n, const int64_t* rowptr, const int32_t* col, const double* K_c,
                   const double* C_c, const double* M_c, double s_re, double s_im, rq_zeig_t** out) {
  return guarded([&] {
    need(s2, "symbolic");
    need(rowptr, "rowptr");
    need(col, "col");
    need(K_c, "K");
    need(C_c, "C");
    need(M_c, "M");
    need(out, "out");
    if (2 * n != s2->S.n) rqb::fail(rqb::errc::dimension, "the ordering must cover the 2n real-equivalent unknowns");
    if (!std::isfinite(s_re) || !std::isfinite(s_im)) rqb::fail(rqb::errc::config, "shift must be finite");
    const int64_t nnz = rowptr[n];
    std::vector<double> qre(nnz), qim(nnz);
    const std::complex<double> sc(s_re, s_im);
    for (int64_t k = 0; k < nnz; ++k) {
      const std::complex<double> kk(K_c[2 * k], K_c[2 * k + 1]), cc(C_c[2 * k], C_c[2 * k + 1]),
          mm(M_c[2 * k], M_c[2 * k + 1]);
      const std::complex<double> q = kk + sc * cc + sc * sc * mm;
      qre[k] = q.real();
      qim[k] = q.imag();
    }
    std::vector<int64_t> rp2;
    std::vector<int32_t> col2;
    std::vector<double> v2;
    complex_equivalent(n, rowptr, col, qre.data(), qim.data(), rp2, col2, v2);
    auto h = std::make_unique<rq_zeig>();
    h->E = std::make_unique<rqb::ZOperatorEngine>(n, rowptr, col, K_c, C_c, M_c, s2->S, s_re, s_im, rp2, col2, v2);
    const double* mats[3] = {K_c, C_c, M_c};
    for (int w = 0; w < 3; ++w) {  // 1-norms (max column sum of |a|; sparse.cpp:38-45)
      std::vector<double> cs(n, 0.0);
      for (int64_t r = 0; r < n; ++r)
        for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) cs[col[k]] += std::hypot(mats[w][2 * k], mats[w][2 * k + 1]);
      h->norms1[w] = cs.empty() ? 0.0 : *std::max_element(cs.begin(), cs.end());
    }
    *out = h.release();
  });
}

int rq_zeig_run(rq_zeig_t* h, int nev, int m, double tol, uint64_t seed, int max_restarts, double* lam_c,
                double* resid, double* vec_c, int32_t* stats) {
  return guarded([&] {
    need(h, "handle");
    need(lam_c, "lam");
    need(resid, "resid");
    std::lock_guard<std::mutex> lock(h->E->fac->mu);
    rqb::ZEigsOptions o;
    o.nev = nev;
    o.m = m;
    o.tol = tol;
    o.seed = seed;
    o.max_restarts = max_restarts > 0 ? max_restarts : 100;
    o.want_vectors = vec_c ? 1 : 0;
    const rqb::ZEigsResult r = rqb::solve_quadratic_complex(*h->E, o, h->norms1);
    for (int i = 0; i < nev; ++i) {
      const bool have = i < static_cast<int>(r.lambda.size());
      lam_c[2 * i] = have ? r.lambda[i].real() : 0.0;
      lam_c[2 * i + 1] = have ? r.lambda[i].imag() : 0.0;
      resid[i] = have ? r.resid[i] : 1.0;
    }
    if (vec_c && !r.vec.empty()) std::memcpy(vec_c, r.vec.data(), sizeof(double) * r.vec.size());
    if (stats) stats[0] = r.cycles, stats[1] = r.nconv;
    if (!r.converged)
      rqb::fail(rqb::errc::solver, "complex solve_quadratic: only " + std::to_string(r.nconv) +
                                       " pairs converged within max_restarts");
  });
}

void rq_zeig_destroy(rq_zeig_t* h) { delete h; }
