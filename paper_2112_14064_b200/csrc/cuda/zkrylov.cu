// SPDX-License-Identifier: Apache-2.0
// Complex shift-invert operator of the linearised pencil (SURVEY.md §8 f4:
// complex shifts and complex pencils, e.g. the conductive EM problem with C =
// -i sigma M_sigma; SPEC.md:408-443 over complex scalars, "Complex shift
// support: Q(s) complex non-symmetric handled by the pivoting LU").
//
// Complex vectors are stored interleaved {re, im} (the reference's cdouble
// layout); a 2N Krylov vector is [v_u (N complex) | v_l (N complex)]. Q(s) =
// K + s C + s^2 M (complex) is factored on the GPU as its real-equivalent 2N
// system (the interleaved layout IS the real-equivalent unknown order), by the
// same multifrontal LU and sweeps as the real path.
//   zspmv_op   t = C v_u + M (s v_u + v_l)       (one pass over the pattern)
//   solve      r_u = -Q(s)^{-1} t                (real-equivalent sweeps)
//   zaxpy      r_l = s r_u + v_u
//   zgemv_t    h = V^H w (conjugated projections, deterministic two-stage sums)
//   zgemv_n    r -= V h
//   zgemm      X = V Q (restart / Ritz vectors)
//   zresidual  ||K u + lam C u + lam^2 M u||^2, ||u||^2 per candidate
#include <cmath>
#include <complex>
#include <vector>

#include "device.cuh"
#include "../host/zeigs.hpp"

namespace rqb {

namespace {

constexpr int kZT = 256;
constexpr int kZBlocks = 592;

int zdiv_up(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

struct z2 {
  double x, y;
};
__device__ __forceinline__ z2 zmul(z2 a, z2 b) { return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__device__ __forceinline__ z2 ld2(const double* p) {
  const double2 v = *reinterpret_cast<const double2*>(p);
  return {v.x, v.y};
}

// y_i = sum_j A_ij x_j (complex), one warp per row
__global__ void zspmv_k(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                        const double* __restrict__ A, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double sr = 0.0, si = 0.0;
  for (int64_t k = rowptr[row] + lane; k < rowptr[row + 1]; k += 32) {
    const z2 a = ld2(A + 2 * k), v = ld2(x + 2 * (int64_t)col[k]);
    const z2 p = zmul(a, v);
    sr += p.x;
    si += p.y;
  }
  sr = warp_sum(sr);
  si = warp_sum(si);
  if (lane == 0) {
    y[2 * row] = sr;
    y[2 * row + 1] = si;
  }
}

// t = C v_u + M (s v_u + v_l)
__global__ void zspmv_op_k(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                           const double* __restrict__ C, const double* __restrict__ M, double sr, double si,
                           const double* __restrict__ vu, const double* __restrict__ vl, double* __restrict__ t) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const z2 s = {sr, si};
  double ar = 0.0, ai = 0.0;
  for (int64_t k = rowptr[row] + lane; k < rowptr[row + 1]; k += 32) {
    const int64_t c = col[k];
    const z2 u = ld2(vu + 2 * c), l = ld2(vl + 2 * c);
    const z2 su = zmul(s, u);
    const z2 cu = zmul(ld2(C + 2 * k), u), mm = zmul(ld2(M + 2 * k), {su.x + l.x, su.y + l.y});
    ar += cu.x + mm.x;
    ai += cu.y + mm.y;
  }
  ar = warp_sum(ar);
  ai = warp_sum(ai);
  if (lane == 0) {
    t[2 * row] = ar;
    t[2 * row + 1] = ai;
  }
}

// r_l = s r_u + v_u (n complex entries)
__global__ void zaxpy_k(int64_t n, double sr, double si, const double* __restrict__ ru, const double* __restrict__ vu,
                        double* __restrict__ rl) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const z2 p = zmul({sr, si}, ld2(ru + 2 * e));
    const z2 v = ld2(vu + 2 * e);
    rl[2 * e] = p.x + v.x;
    rl[2 * e + 1] = p.y + v.y;
  }
}

// part[(b * k + i) * 2 + {0,1}] = sum over block b's entries of conj(V_i) w
// (len complex entries per vector, vectors at stride ldv doubles)
__global__ void __launch_bounds__(kZT) zgemv_t_part(const double* __restrict__ V, int k, int64_t ldv, int64_t len,
                                                  const double* __restrict__ w, double* __restrict__ part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t per = (len + gridDim.x - 1) / gridDim.x;
  const int64_t e0 = blockIdx.x * per, e1 = min(len, e0 + per);
  for (int i = warp; i < k; i += kZT / 32) {
    const double* v = V + (int64_t)i * ldv;
    double sr = 0.0, si = 0.0;
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const z2 a = ld2(v + 2 * e), b = ld2(w + 2 * e);
      sr += a.x * b.x + a.y * b.y;  // conj(a) b
      si += a.x * b.y - a.y * b.x;
    }
    sr = warp_sum(sr);
    si = warp_sum(si);
    if (lane == 0) {
      part[((int64_t)blockIdx.x * k + i) * 2] = sr;
      part[((int64_t)blockIdx.x * k + i) * 2 + 1] = si;
    }
  }
}

__global__ void zreduce_k(const double* __restrict__ part, int nb, int k, double* __restrict__ h) {
  const int i = blockIdx.x, lane = threadIdx.x;
  double sr = 0.0, si = 0.0;
  for (int b = lane; b < nb; b += 32) {
    sr += part[((int64_t)b * k + i) * 2];
    si += part[((int64_t)b * k + i) * 2 + 1];
  }
  sr = warp_sum(sr);
  si = warp_sum(si);
  if (lane == 0) {
    h[2 * i] = sr;
    h[2 * i + 1] = si;
  }
}

// r -= sum_i h_i V_i
__global__ void zgemv_n_k(const double* __restrict__ V, int k, int64_t ldv, int64_t len, const double* __restrict__ h,
                          double* __restrict__ r) {
  extern __shared__ double hs[];
  for (int i = threadIdx.x; i < 2 * k; i += blockDim.x) hs[i] = h[i];
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len; e += (int64_t)gridDim.x * blockDim.x) {
    double sr = 0.0, si = 0.0;
    for (int i = 0; i < k; ++i) {
      const z2 p = zmul({hs[2 * i], hs[2 * i + 1]}, ld2(V + (int64_t)i * ldv + 2 * e));
      sr += p.x;
      si += p.y;
    }
    r[2 * e] -= sr;
    r[2 * e + 1] -= si;
  }
}

// X[:, c] = sum_t V[:, t] Q[t + c ldq] (complex), c < nc
__global__ void zgemm_k(const double* __restrict__ V, int k, int64_t ldv, int64_t len, const double* __restrict__ Q,
                        int ldq, int nc, double* __restrict__ X, int64_t ldx) {
  const int c = blockIdx.y;
  extern __shared__ double qs[];
  for (int t = threadIdx.x; t < 2 * k; t += blockDim.x) qs[t] = Q[2 * ((int64_t)c * ldq) + t];
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len; e += (int64_t)gridDim.x * blockDim.x) {
    double sr = 0.0, si = 0.0;
    for (int t = 0; t < k; ++t) {
      const z2 p = zmul({qs[2 * t], qs[2 * t + 1]}, ld2(V + (int64_t)t * ldv + 2 * e));
      sr += p.x;
      si += p.y;
    }
    X[(int64_t)c * ldx + 2 * e] = sr;
    X[(int64_t)c * ldx + 2 * e + 1] = si;
  }
}

// per block b: partial of ||r||^2 (r = x - s y for real-valued dots of
// interleaved vectors): part[b] = sum x . y over the block's doubles
__global__ void __launch_bounds__(kZT) rdot_k(const double* __restrict__ x, const double* __restrict__ y, int64_t len2,
                                            double* __restrict__ part) {
  __shared__ double sh[kZT / 32];
  double s = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len2; e += (int64_t)gridDim.x * blockDim.x)
    s += x[e] * y[e];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kZT / 32; ++w) t += sh[w];
    part[blockIdx.x] = t;
  }
}

// beta = sqrt(sum part); v = r / beta, bv = w / beta (2 len doubles each)
__global__ void znormalize_k(const double* __restrict__ part, int nb, const double* __restrict__ r,
                             const double* __restrict__ w, int64_t len2, double* __restrict__ beta_out,
                             double* __restrict__ v, double* __restrict__ bv) {
  __shared__ double beta_s;
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int b = threadIdx.x; b < nb; b += 32) s += part[b];
    s = warp_sum(s);
    if (threadIdx.x == 0) {
      beta_s = sqrt(fmax(s, 0.0));
      if (blockIdx.x == 0 && beta_out) *beta_out = beta_s;
    }
  }
  __syncthreads();
  const double inv = beta_s > 0.0 ? 1.0 / beta_s : 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len2; e += (int64_t)gridDim.x * blockDim.x) {
    v[e] = r[e] * inv;
    bv[e] = w[e] * inv;
  }
}

// q = K u + lam C u + lam^2 M u for candidate c (u: n complex at X + c ldx),
// partials of ||q||^2 and ||u||^2
__global__ void __launch_bounds__(kZT) zresidual_k(int64_t n, const int64_t* __restrict__ rowptr,
                                                 const int32_t* __restrict__ col, const double* __restrict__ K,
                                                 const double* __restrict__ C, const double* __restrict__ M,
                                                 const double* __restrict__ X, int64_t ldx,
                                                 const double* __restrict__ lam, double* __restrict__ part) {
  __shared__ double sq[kZT / 32], su[kZT / 32];
  const int c = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* u = X + (int64_t)c * ldx;
  const z2 l = {lam[2 * c], lam[2 * c + 1]};
  const z2 l2 = zmul(l, l);
  double aq = 0.0, au = 0.0;
  for (int64_t row = blockIdx.x * (int64_t)(kZT / 32) + warp; row < n; row += (int64_t)gridDim.x * (kZT / 32)) {
    double kr = 0, ki = 0, cr = 0, ci = 0, mr = 0, mi = 0;
    for (int64_t k = rowptr[row] + lane; k < rowptr[row + 1]; k += 32) {
      const z2 x = ld2(u + 2 * (int64_t)col[k]);
      const z2 a = zmul(ld2(K + 2 * k), x), b = zmul(ld2(C + 2 * k), x), d = zmul(ld2(M + 2 * k), x);
      kr += a.x, ki += a.y, cr += b.x, ci += b.y, mr += d.x, mi += d.y;
    }
    kr = warp_sum(kr), ki = warp_sum(ki), cr = warp_sum(cr), ci = warp_sum(ci), mr = warp_sum(mr), mi = warp_sum(mi);
    const z2 lc = zmul(l, {cr, ci}), lm = zmul(l2, {mr, mi});
    const double qr = kr + lc.x + lm.x, qi = ki + lc.y + lm.y;
    const z2 ux = ld2(u + 2 * row);
    aq += qr * qr + qi * qi;
    au += ux.x * ux.x + ux.y * ux.y;
  }
  if (lane == 0) sq[warp] = aq, su[warp] = au;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int w = 0; w < kZT / 32; ++w) s0 += sq[w], s1 += su[w];
    part[((int64_t)c * gridDim.x + blockIdx.x) * 2] = s0;
    part[((int64_t)c * gridDim.x + blockIdx.x) * 2 + 1] = s1;
  }
}

}  // namespace

ZOperatorEngine::ZOperatorEngine(int64_t n_, const int64_t* rowptr, const int32_t* col, const double* K,
                                 const double* C, const double* M, const Symbolic& s2, double sr, double si,
                                 const std::vector<int64_t>& rp2, const std::vector<int32_t>& col2,
                                 const std::vector<double>& q2)
    : n(n_), s_re(sr), s_im(si) {
  nnz = rowptr[n];
  fac = std::make_unique<FactorEngine>(s2, 2 * n, rp2.data(), col2.data(), q2.data());
  stream = fac->stream;
  d_rowptr.upload(rowptr, sizeof(int64_t) * (n + 1), stream);
  d_col.upload(col, sizeof(int32_t) * std::max<int64_t>(nnz, 1), stream);
  d_K.upload(K, sizeof(double) * 2 * nnz, stream);
  d_C.upload(C, sizeof(double) * 2 * nnz, stream);
  d_M.upload(M, sizeof(double) * 2 * nnz, stream);
  d_t.alloc(sizeof(double) * 2 * n);
  d_part.alloc(sizeof(double) * kZBlocks * 2 * 520);
  RQB_CUDA(cudaStreamSynchronize(stream));
  fac->factor();
}

void ZOperatorEngine::spmv(int which, const double* x, double* y) {
  const double* A = which == 0 ? d_K.as<double>() : which == 1 ? d_C.as<double>() : d_M.as<double>();
  zspmv_k<<<zdiv_up(n * 32, 256), 256, 0, stream>>>(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(), A, x, y);
  ++launches;
}

void ZOperatorEngine::apply(const double* v, double* r) {
  double* t = d_t.as<double>();
  zspmv_op_k<<<zdiv_up(n * 32, 256), 256, 0, stream>>>(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(),
                                                       d_C.as<double>(), d_M.as<double>(), s_re, s_im, v, v + 2 * n,
                                                       t);
  rqb_solve_enqueue(*fac, t, r, -1.0, nullptr, 0.0, nullptr);  // the 2n real-equivalent unknowns
  zaxpy_k<<<std::min(zdiv_up(n, 256), 148 * 8), 256, 0, stream>>>(n, s_re, s_im, r, v, r + 2 * n);
  launches += 2 + fac->launches_solve;
}

void ZOperatorEngine::bvec(const double* r, double* w) {
  RQB_CUDA(cudaMemcpyAsync(w, r, sizeof(double) * 2 * n, cudaMemcpyDeviceToDevice, stream));
  spmv(2, r + 2 * n, w + 2 * n);
}

void ZOperatorEngine::gemv_t(const double* V, int k, int64_t ldv, const double* w, double* h) {
  if (k <= 0) return;
  if (k > 520) fail(errc::config, "Krylov dimension above 520");
  zgemv_t_part<<<kZBlocks, kZT, 0, stream>>>(V, k, ldv, 2 * n, w, d_part.as<double>());
  zreduce_k<<<k, 32, 0, stream>>>(d_part.as<double>(), kZBlocks, k, h);
  launches += 2;
}

void ZOperatorEngine::gemv_n(const double* V, int k, int64_t ldv, const double* h, double* r) {
  if (k <= 0) return;
  zgemv_n_k<<<std::min(zdiv_up(2 * n, 256), 148 * 8), 256, sizeof(double) * 2 * k, stream>>>(V, k, ldv, 2 * n, h, r);
  ++launches;
}

void ZOperatorEngine::bnorm_normalize(const double* r, const double* w, double* beta_out, double* v, double* bv) {
  rdot_k<<<kZBlocks, kZT, 0, stream>>>(r, w, 4 * n, d_part.as<double>());
  znormalize_k<<<std::min(zdiv_up(4 * n, 256), 148 * 8), 256, 0, stream>>>(d_part.as<double>(), kZBlocks, r, w,
                                                                          4 * n, beta_out, v, bv);
  launches += 2;
}

void ZOperatorEngine::combine(const double* V, int k, int64_t ldv, int64_t len, const double* Q, int ldq, int nc,
                              double* X, int64_t ldx) {
  if (k <= 0 || nc <= 0) return;
  dim3 grid(std::min(zdiv_up(len, 256), 148 * 2), nc);
  zgemm_k<<<grid, 256, sizeof(double) * 2 * k, stream>>>(V, k, ldv, len, Q, ldq, nc, X, ldx);
  ++launches;
}

void ZOperatorEngine::residuals(const double* X, int64_t ldx, int nc, const double* lam_host, double* out_host) {
  if (nc <= 0) return;
  const int nbx = kZBlocks;
  if (d_res.bytes < sizeof(double) * (2 * static_cast<size_t>(nc) * nbx + 2 * nc))
    d_res.alloc(sizeof(double) * (2 * static_cast<size_t>(nc) * nbx + 2 * nc));
  double* part = d_res.as<double>();
  double* dl = part + 2 * static_cast<size_t>(nc) * nbx;
  RQB_CUDA(cudaMemcpyAsync(dl, lam_host, sizeof(double) * 2 * nc, cudaMemcpyHostToDevice, stream));
  zresidual_k<<<dim3(nbx, nc), kZT, 0, stream>>>(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(), d_K.as<double>(),
                                                 d_C.as<double>(), d_M.as<double>(), X, ldx, dl, part);
  std::vector<double> h(2 * static_cast<size_t>(nc) * nbx);
  RQB_CUDA(cudaMemcpyAsync(h.data(), part, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, stream));
  RQB_CUDA(cudaStreamSynchronize(stream));
  ++launches;
  for (int c = 0; c < nc; ++c) {
    double a = 0.0, b = 0.0;
    for (int blk = 0; blk < nbx; ++blk) a += h[(static_cast<size_t>(c) * nbx + blk) * 2], b += h[(static_cast<size_t>(c) * nbx + blk) * 2 + 1];
    out_host[2 * c] = a;
    out_host[2 * c + 1] = b;
  }
}

}  // namespace rqb
