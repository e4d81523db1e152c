// SPDX-License-Identifier: Apache-2.0
// Shift-invert operator and Krylov kernels (real FP64, device resident).
//
//   spmv_csr        y = A x, one warp per row (kern::spmv_csr, kernels.cpp:44-56)
//   spmv_op         t = C v_u + M (s v_u + v_l): the three products of
//                   apply_operator in one pass over the shared
//                   pattern (col[] read once, two value streams)
//   gemv_t_part     h = V^T w: CGS2 projection (kern::dotc, kernels.cpp:23-32,
//                   fused over all basis vectors; one pass over V), block
//                   partials + fixed-order final reduction (deterministic)
//   gemv_n          r -= V h (kern::axpy, kernels.cpp:19-21, fused)
//   normalize       B-norm and v = r / ||r||_B (kern::nrm2sq/scal fused)
//   combine         V Q (Krylov-Schur restart / Ritz vectors): cuBLAS DGEMM
//   ritz_residual   ||Q(lambda_c) x_c||^2, ||x_c||^2 for a batch of Ritz vectors
//                   (row-major, from one DGEMM): SpMM over K, C, M
#include <cmath>
#include <cstring>
#include <vector>


#include "device.cuh"

namespace rqb {

namespace {

constexpr int kRedBlocks = 592;  // 4 x 148 SMs: partial-sum blocks of the reductions
constexpr int kRedThreads = 256;

int div_up(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
  return s;  // valid in thread 0
}

}  // namespace

__global__ void spmv_csr_k(int64_t n, const int64_t* __restrict__ rowptr,
                           const int32_t* __restrict__ col, const double* __restrict__ val,
                           const double* __restrict__ x, double* __restrict__ y) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double s = 0.0;
  for (int64_t k = rowptr[row] + lane; k < rowptr[row + 1]; k += 32) s += val[k] * x[col[k]];
  s = warp_sum(s);
  if (lane == 0) y[row] = s;
}

__global__ void spmv_op_k(int64_t n, const int64_t* __restrict__ rowptr,
                          const int32_t* __restrict__ col, const double* __restrict__ Cv,
                          const double* __restrict__ Mv, double sigma,
                          const double* __restrict__ vu, const double* __restrict__ vl,
                          double* __restrict__ t) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double s = 0.0;
  for (int64_t k = rowptr[row] + lane; k < rowptr[row + 1]; k += 32) {
    const int c = col[k];
    const double xu = vu[c];
    s += Cv[k] * xu + Mv[k] * (sigma * xu + vl[c]);
  }
  s = warp_sum(s);
  if (lane == 0) t[row] = s;
}

// Version 2 of the CSR products (RQB_SPMV=1 selects the version above): LPR
// lanes per row (32 / LPR rows per warp, fewer idle lane slots on short
// rows), and each lane issues the (col, value) loads of U entries (k, k + LPR,
// ..., k + LPR (U - 1)) before any gather, so U entries per lane are in
// flight instead of one; the pattern and values are read once per product,
// so they are loaded with the streaming hint (evict-first) and the gathered
// vector keeps its L2 lines.
template <int U, int LPR>
__global__ void __launch_bounds__(256) spmv_csr_k2(int64_t n, const int64_t* __restrict__ rowptr,
                                                  const int32_t* __restrict__ col, const double* __restrict__ val,
                                                  const double* __restrict__ x, double* __restrict__ y) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / LPR;
  const int sl = threadIdx.x & (LPR - 1);
  double s = 0.0;
  if (row < n) {
    const int64_t e = __ldg(&rowptr[row + 1]);
    for (int64_t k0 = __ldg(&rowptr[row]) + sl; k0 < e; k0 += LPR * U) {
      int c[U];
      double a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t k = k0 + LPR * u;
        c[u] = k < e ? __ldcs(&col[k]) : -1;
        a[u] = k < e ? __ldcs(&val[k]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c[u] >= 0) s += a[u] * __ldg(&x[c[u]]);
    }
  }
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (row < n && sl == 0) y[row] = s;
}

template <int U, int LPR>
__global__ void __launch_bounds__(256) spmv_op_k2(int64_t n, const int64_t* __restrict__ rowptr,
                                                 const int32_t* __restrict__ col, const double* __restrict__ Cv,
                                                 const double* __restrict__ Mv, double sigma,
                                                 const double* __restrict__ vu, const double* __restrict__ vl,
                                                 double* __restrict__ t) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / LPR;
  const int sl = threadIdx.x & (LPR - 1);
  double s = 0.0;
  if (row < n) {
    const int64_t e = __ldg(&rowptr[row + 1]);
    for (int64_t k0 = __ldg(&rowptr[row]) + sl; k0 < e; k0 += LPR * U) {
      int c[U];
      double cv[U], mv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t k = k0 + LPR * u;
        const bool ok = k < e;
        c[u] = ok ? __ldcs(&col[k]) : -1;
        cv[u] = ok ? __ldcs(&Cv[k]) : 0.0;
        mv[u] = ok ? __ldcs(&Mv[k]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c[u] >= 0) {
          const double xu = __ldg(&vu[c[u]]);
          s += cv[u] * xu + mv[u] * (sigma * xu + __ldg(&vl[c[u]]));
        }
    }
  }
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (row < n && sl == 0) t[row] = s;
}

// part[b * k + i] = sum over block b's slice of V[i] . w  (w given as two halves)
// part[b*k + i] = V[i][chunk b] . w[chunk b]: the block stages its chunk of
// w in shared memory once; each warp then owns basis vectors i = warp (mod 8),
// four at a time, streaming their contiguous chunk segments (16 independent
// loads in flight per lane) and reducing with shuffles only.
__global__ void __launch_bounds__(kRedThreads) gemv_t_part(const double* __restrict__ V, int k,
                                                         int64_t n2, const double* __restrict__ wu,
                                                         const double* __restrict__ wl, int64_t n,
                                                         int64_t chunk, double* __restrict__ part) {
  extern __shared__ double xs[];
  const int64_t e0 = blockIdx.x * chunk;
  const int len = static_cast<int>(min(chunk, n2 - e0));
  for (int t = threadIdx.x; t < len; t += kRedThreads) {
    const int64_t e = e0 + t;
    xs[t] = e < n ? wu[e] : wl[e - n];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kW = kRedThreads / 32, kV = 4;  // basis vectors per warp pass
  for (int i = warp; i < k; i += kV * kW) {
    const double* vp[kV];
#pragma unroll
    for (int q = 0; q < kV; ++q) vp[q] = V + (int64_t)(i + q * kW < k ? i + q * kW : i) * n2 + e0;
    double s0[kV], s1[kV];
#pragma unroll
    for (int q = 0; q < kV; ++q) s0[q] = s1[q] = 0.0;
    int t = lane;
    for (; t + 32 * 3 < len; t += 32 * 4) {  // 16 loads in flight per lane
      double a[kV][4];
#pragma unroll
      for (int q = 0; q < kV; ++q)
#pragma unroll
        for (int u = 0; u < 4; ++u) a[q][u] = vp[q][t + 32 * u];
      const double x0 = xs[t], x1 = xs[t + 32], x2 = xs[t + 64], x3 = xs[t + 96];
#pragma unroll
      for (int q = 0; q < kV; ++q) {
        s0[q] += a[q][0] * x0 + a[q][2] * x2;
        s1[q] += a[q][1] * x1 + a[q][3] * x3;
      }
    }
    for (; t < len; t += 32)
#pragma unroll
      for (int q = 0; q < kV; ++q) s0[q] += vp[q][t] * xs[t];
#pragma unroll
    for (int q = 0; q < kV; ++q) {
      const double sq = warp_sum(s0[q] + s1[q]);
      if (lane == 0 && i + q * kW < k) part[(int64_t)blockIdx.x * k + i + q * kW] = sq;
    }
  }
}

// h[i] = sum_b part[b*k + i]  (fixed order), optionally hacc[i] += h[i]
__global__ void reduce_parts(const double* __restrict__ part, int nb, int k, double* __restrict__ h,
                             double* __restrict__ hacc) {
  const int i = blockIdx.x;
  const int lane = threadIdx.x;
  double s = 0.0;
  for (int b = lane; b < nb; b += 32) s += part[(int64_t)b * k + i];
  s = warp_sum(s);
  if (lane == 0) {
    h[i] = s;
    if (hacc) hacc[i] += s;
  }
}

// r[e] -= sum_i V[i ldv + e] h[i], e < len
__global__ void gemv_n_k(const double* __restrict__ V, int k, int64_t ldv, int64_t len,
                         const double* __restrict__ h, double* __restrict__ r) {
  extern __shared__ double hs[];
  for (int i = threadIdx.x; i < k; i += blockDim.x) hs[i] = h[i];
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < k; ++i) s += V[(int64_t)i * ldv + e] * hs[i];
    r[e] -= s;
  }
}

// part[b] = sum over slice of x.y (x, y given as halves: xu|xl and yu|yl)
__global__ void __launch_bounds__(kRedThreads) dot_part(const double* __restrict__ xu,
                                                      const double* __restrict__ xl,
                                                      const double* __restrict__ yu,
                                                      const double* __restrict__ yl, int64_t n,
                                                      int64_t n2, double* __restrict__ part) {
  __shared__ double sh[kRedThreads / 32];
  double s = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n2;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double a = e < n ? xu[e] : xl[e - n];
    const double b = e < n ? yu[e] : yl[e - n];
    s += a * b;
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// beta = sqrt(sum parts) -> *beta_out; v = r / beta
__global__ void normalize_k(const double* __restrict__ part, int nb, const double* __restrict__ r,
                            int64_t n2, double* __restrict__ beta_out, double* __restrict__ v) {
  __shared__ double beta_s;
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int b = threadIdx.x; b < nb; b += 32) s += part[b];
    s = warp_sum(s);
    if (threadIdx.x == 0) {
      const double beta = sqrt(fmax(s, 0.0));
      beta_s = beta;
      if (blockIdx.x == 0 && beta_out) *beta_out = beta;
    }
  }
  __syncthreads();
  const double inv = beta_s > 0.0 ? 1.0 / beta_s : 0.0;
  if (v)
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n2;
         e += (int64_t)gridDim.x * blockDim.x)
      v[e] = r[e] * inv;
}

__global__ void sum_parts(const double* __restrict__ part, int nb, double* __restrict__ out) {
  double s = 0.0;
  for (int b = threadIdx.x; b < nb; b += 32) s += part[b];
  s = warp_sum(s);
  if (threadIdx.x == 0) *out = s;
}

// Vout[c][e] = sum_i V[i][e] Q[i + c*ldq], c in [c0, c0+8)

// per-row complex pencil residual of (lambda, u = ur + i ui); parts of
// ||Q(lambda)u||^2 (out[b]) and ||u||^2 (out[nb + b])


// Pencil residuals of a batch of Ritz vectors held ROW-major (X[e * ldx + 2c]
// = Re x_c[e], X[e * ldx + 2c + 1] = Im x_c[e], e < 2n): an SpMM over the
// shared pattern of K, C, M. Lane l owns candidates c0 + l and c0 + 32 + l of
// the block's 64; the warp loads 32 nonzeros (col, K, C, M) coalesced and
// broadcasts them, each candidate gathering one 16-byte {re, im} pair per
// nonzero (the 64 candidates of a nonzero are one contiguous 1 KiB row).
// part[(2c + {0,1}) * gridDim.x + block] = partial {||Q(lambda_c) u_c||^2, ||u_c||^2}.
__global__ void __launch_bounds__(kRedThreads) ritz_residual_k(
    int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
    const double* __restrict__ K, const double* __restrict__ C, const double* __restrict__ M,
    const double* __restrict__ X, int ldx, int nc, const double* __restrict__ lam,
    const int* __restrict__ blk, double* __restrict__ part) {
  constexpr int kW = kRedThreads / 32;
  __shared__ double sred[kW][16][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double lr[2], li[2], sr[2], si[2], acc[2] = {0.0, 0.0}, accu[2] = {0.0, 0.0};
  double rq[2][6] = {{0, 0, 0, 0, 0, 0}, {0, 0, 0, 0, 0, 0}};  // u^H K u, u^H C u, u^H M u (re, im)
  const double* xb[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = min(nc - 1, (int)blockIdx.y * 64 + 32 * h + lane);
    lr[h] = lam[2 * c];
    li[h] = lam[2 * c + 1];
    sr[h] = lr[h] * lr[h] - li[h] * li[h];
    si[h] = 2.0 * lr[h] * li[h];
    xb[h] = X + (int64_t)blk[c] * n * ldx + 2 * c;
  }
  for (int64_t row = blockIdx.x * (int64_t)kW + warp; row < n; row += (int64_t)gridDim.x * kW) {
    double a[2][6];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int t = 0; t < 6; ++t) a[h][t] = 0.0;
    const int64_t k0 = rowptr[row], k1 = rowptr[row + 1];
    for (int64_t kb = k0; kb < k1; kb += 32) {
      const int cnt = static_cast<int>(k1 - kb < 32 ? k1 - kb : 32);
      int jl = 0;
      double kl = 0.0, cl = 0.0, ml = 0.0;
      if (lane < cnt) {
        jl = col[kb + lane];
        kl = K[kb + lane];
        cl = C[kb + lane];
        ml = M[kb + lane];
      }
#pragma unroll 4
      for (int t = 0; t < cnt; ++t) {
        const int64_t j = __shfl_sync(0xffffffffu, jl, t);
        const double kv = __shfl_sync(0xffffffffu, kl, t);
        const double cv = __shfl_sync(0xffffffffu, cl, t);
        const double mv = __shfl_sync(0xffffffffu, ml, t);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double2 x = *reinterpret_cast<const double2*>(xb[h] + j * ldx);
          a[h][0] += kv * x.x;
          a[h][1] += kv * x.y;
          a[h][2] += cv * x.x;
          a[h][3] += cv * x.y;
          a[h][4] += mv * x.x;
          a[h][5] += mv * x.y;
        }
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double re = a[h][0] + (lr[h] * a[h][2] - li[h] * a[h][3]) + (sr[h] * a[h][4] - si[h] * a[h][5]);
      const double im = a[h][1] + (lr[h] * a[h][3] + li[h] * a[h][2]) + (sr[h] * a[h][5] + si[h] * a[h][4]);
      const double2 u = *reinterpret_cast<const double2*>(xb[h] + row * ldx);
      acc[h] += re * re + im * im;
      accu[h] += u.x * u.x + u.y * u.y;
#pragma unroll
      for (int t = 0; t < 3; ++t) {  // conj(u) (A u): the quadratic Rayleigh quotient's coefficients
        rq[h][2 * t] += u.x * a[h][2 * t] + u.y * a[h][2 * t + 1];
        rq[h][2 * t + 1] += u.x * a[h][2 * t + 1] - u.y * a[h][2 * t];
      }
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    sred[warp][8 * h][lane] = acc[h];
    sred[warp][8 * h + 1][lane] = accu[h];
#pragma unroll
    for (int t = 0; t < 6; ++t) sred[warp][8 * h + 2 + t][lane] = rq[h][t];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = (int)blockIdx.y * 64 + 32 * h + lane;
      double sv[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        sv[t] = 0.0;
        for (int w = 0; w < kW; ++w) sv[t] += sred[w][8 * h + t][lane];
      }
      if (c < nc) {
        part[(int64_t)(2 * c) * gridDim.x + blockIdx.x] = sv[0];
        part[(int64_t)(2 * c + 1) * gridDim.x + blockIdx.x] = sv[1];
        // rows [2 nc, 8 nc): the Rayleigh-quotient coefficients, 6 per candidate
#pragma unroll
        for (int t = 0; t < 6; ++t) part[(int64_t)(2 * nc + 6 * c + t) * gridDim.x + blockIdx.x] = sv[2 + t];
      }
    }
  }
}

// out[j] = X[(blk_c n + j) * ldx + 2c + part] (one Ritz vector of a row-major
// batch back to a contiguous vector; part 0 real, 1 imaginary)
__global__ void ritz_extract_k(const double* __restrict__ X, int ldx, int64_t n, const int* __restrict__ blk,
                               int c, int part_im, double* __restrict__ out) {
  const double* src = X + (int64_t)blk[c] * n * ldx + 2 * c + part_im;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    out[j] = src[j * ldx];
}

// ---- block Krylov-Schur: kernels over a block of bs <= 8 vectors ----

// Xi[e * KB + j] = V[j * ldv + e] (j < bs; zero for bs <= j < KB), e < 2n:
// the block row-interleaved, so a gather of one column index reads all the
// block's values in one 32- or 64-byte segment
template <int KB>
__global__ void interleave_k(const double* __restrict__ V, int64_t ldv, int64_t n2, int bs, double* __restrict__ Xi) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n2; e += (int64_t)gridDim.x * blockDim.x) {
    double v[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j) v[j] = j < bs ? V[j * ldv + e] : 0.0;
    double2* o = reinterpret_cast<double2*>(Xi + e * KB);
#pragma unroll
    for (int q = 0; q < KB / 2; ++q) o[q] = make_double2(v[2 * q], v[2 * q + 1]);
  }
}

// Ti[row * KB + j] = C v_u^j + M (s v_u^j + v_l^j) from the interleaved block
// Xi (upper rows [0, n), lower [n, 2n)): one pass over the shared pattern
// (col, C, M read once for all KB vectors), 2 x KB / 2 double2 gathers per nonzero
template <int KB>
__global__ void spmm_op_k(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                          const double* __restrict__ Cv, const double* __restrict__ Mv, double sigma,
                          const double* __restrict__ Xi, double* __restrict__ Ti) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double s[KB];
#pragma unroll
  for (int j = 0; j < KB; ++j) s[j] = 0.0;
  for (int64_t k = rowptr[row] + lane; k < rowptr[row + 1]; k += 32) {
    const int64_t c = col[k];
    const double cv = Cv[k], mv = Mv[k];
    const double2* xu = reinterpret_cast<const double2*>(Xi + c * KB);
    const double2* xl = reinterpret_cast<const double2*>(Xi + (n + c) * KB);
#pragma unroll
    for (int q = 0; q < KB / 2; ++q) {
      const double2 u = xu[q], l = xl[q];
      s[2 * q] += cv * u.x + mv * (sigma * u.x + l.x);
      s[2 * q + 1] += cv * u.y + mv * (sigma * u.y + l.y);
    }
  }
#pragma unroll
  for (int j = 0; j < KB; ++j) s[j] = warp_sum(s[j]);
  if (lane == 0) {
    double2* o = reinterpret_cast<double2*>(Ti + row * KB);
#pragma unroll
    for (int q = 0; q < KB / 2; ++q) o[q] = make_double2(s[2 * q], s[2 * q + 1]);
  }
}

// Y[j * ldy + row] = sum_k A[row, k] Xi[col_k * KB + j], j < w (interleaved
// input, column-major output): one pass over the pattern for the w vectors
template <int KB>
__global__ void spmm_csr_k(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                           const double* __restrict__ val, const double* __restrict__ Xi, int w,
                           double* __restrict__ Y, int64_t ldy) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double s[KB];
#pragma unroll
  for (int j = 0; j < KB; ++j) s[j] = 0.0;
  for (int64_t k = rowptr[row] + lane; k < rowptr[row + 1]; k += 32) {
    const double a = val[k];
    const double2* x = reinterpret_cast<const double2*>(Xi + (int64_t)col[k] * KB);
#pragma unroll
    for (int q = 0; q < KB / 2; ++q) {
      const double2 t = x[q];
      s[2 * q] += a * t.x;
      s[2 * q + 1] += a * t.y;
    }
  }
#pragma unroll
  for (int j = 0; j < KB; ++j) {
    const double t = warp_sum(s[j]);
    if (lane == 0 && j < w) Y[j * ldy + row] = t;
  }
}

// 32-byte read-only gather (one LDG.E.256: a whole 4-wide row of an
// interleaved block in one sector access instead of two 16-byte loads)
__device__ __forceinline__ void ldg4(const double* p, double* v) {
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}

// Version 2 of the two block products (see spmv_op_k2): U entries per lane
// in flight, streaming loads of the pattern and values, 32-byte gathers of
// the interleaved rows.
template <int KB, int U, int LPR>
__global__ void __launch_bounds__(256) spmm_op_k2(int64_t n, const int64_t* __restrict__ rowptr,
                                                 const int32_t* __restrict__ col, const double* __restrict__ Cv,
                                                 const double* __restrict__ Mv, double sigma,
                                                 const double* __restrict__ Xi, double* __restrict__ Ti) {
  // LPR lanes per row (32 / LPR rows per warp): fewer idle lane slots on
  // short rows; every lane reaches the shuffles (no early exit)
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / LPR;
  const int sl = threadIdx.x & (LPR - 1);
  double s[KB];
#pragma unroll
  for (int j = 0; j < KB; ++j) s[j] = 0.0;
  if (row < n) {
    const int64_t e = __ldg(&rowptr[row + 1]);
    for (int64_t k0 = __ldg(&rowptr[row]) + sl; k0 < e; k0 += LPR * U) {
      int c[U];
      double cv[U], mv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t k = k0 + LPR * u;
        const bool ok = k < e;
        c[u] = ok ? __ldcs(&col[k]) : -1;
        cv[u] = ok ? __ldcs(&Cv[k]) : 0.0;
        mv[u] = ok ? __ldcs(&Mv[k]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c[u] >= 0) {
          double a[KB], l[KB];
#pragma unroll
          for (int q = 0; q < KB / 4; ++q) {
            ldg4(Xi + (int64_t)c[u] * KB + 4 * q, a + 4 * q);
            ldg4(Xi + (n + c[u]) * KB + 4 * q, l + 4 * q);
          }
#pragma unroll
          for (int j = 0; j < KB; ++j) s[j] += cv[u] * a[j] + mv[u] * (sigma * a[j] + l[j]);
        }
    }
  }
#pragma unroll
  for (int j = 0; j < KB; ++j)
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) s[j] += __shfl_xor_sync(0xffffffffu, s[j], o);
  if (row < n && sl == 0) {
    double2* o = reinterpret_cast<double2*>(Ti + row * KB);
#pragma unroll
    for (int q = 0; q < KB / 2; ++q) o[q] = make_double2(s[2 * q], s[2 * q + 1]);
  }
}

template <int KB, int U, int LPR>
__global__ void __launch_bounds__(256) spmm_csr_k2(int64_t n, const int64_t* __restrict__ rowptr,
                                                  const int32_t* __restrict__ col, const double* __restrict__ val,
                                                  const double* __restrict__ Xi, int w, double* __restrict__ Y,
                                                  int64_t ldy) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / LPR;
  const int sl = threadIdx.x & (LPR - 1);
  double s[KB];
#pragma unroll
  for (int j = 0; j < KB; ++j) s[j] = 0.0;
  if (row < n) {
    const int64_t e = __ldg(&rowptr[row + 1]);
    for (int64_t k0 = __ldg(&rowptr[row]) + sl; k0 < e; k0 += LPR * U) {
      int c[U];
      double a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t k = k0 + LPR * u;
        c[u] = k < e ? __ldcs(&col[k]) : -1;
        a[u] = k < e ? __ldcs(&val[k]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c[u] >= 0) {
          double x[KB];
#pragma unroll
          for (int q = 0; q < KB / 4; ++q) ldg4(Xi + (int64_t)c[u] * KB + 4 * q, x + 4 * q);
#pragma unroll
          for (int j = 0; j < KB; ++j) s[j] += a[u] * x[j];
        }
    }
  }
#pragma unroll
  for (int j = 0; j < KB; ++j) {
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) s[j] += __shfl_xor_sync(0xffffffffu, s[j], o);
    if (row < n && sl == 0 && j < w) Y[j * ldy + row] = s[j];
  }
}

namespace {

int spmv_version() {
  static const int v = std::getenv("RQB_SPMV") ? std::atoi(std::getenv("RQB_SPMV")) : 2;
  return v;
}

// Version 2 launch shapes (measured at cfg4_riga, ~68 nonzeros per row): 8
// lanes per row with 5 entries in flight per lane for the single-vector and
// width-4 products, 4 lanes per row for width 8 (32 lanes x 3: 0.205 / 0.416 /
// 0.842 ms; 16 x 5: 0.174 / 0.298 / 0.629; 8 x 5: 0.172 / 0.263 / 0.590;
// 4 x 5: - / 0.269 / 0.513 for the operator SpMV / width-4 / width-8 SpMM)
void launch_spmv_csr(int64_t n, const int64_t* rp, const int32_t* col, const double* val, const double* x, double* y,
                     cudaStream_t st) {
  if (spmv_version() == 1)
    spmv_csr_k<<<div_up(n * 32, 256), 256, 0, st>>>(n, rp, col, val, x, y);
  else
    spmv_csr_k2<5, 8><<<div_up(n * 8, 256), 256, 0, st>>>(n, rp, col, val, x, y);
}

void launch_spmv_op(int64_t n, const int64_t* rp, const int32_t* col, const double* Cv, const double* Mv,
                    double sigma, const double* vu, const double* vl, double* t, cudaStream_t st) {
  if (spmv_version() == 1)
    spmv_op_k<<<div_up(n * 32, 256), 256, 0, st>>>(n, rp, col, Cv, Mv, sigma, vu, vl, t);
  else
    spmv_op_k2<5, 8><<<div_up(n * 8, 256), 256, 0, st>>>(n, rp, col, Cv, Mv, sigma, vu, vl, t);
}

template <int KB>
void launch_spmm_op(int64_t n, const int64_t* rp, const int32_t* col, const double* Cv, const double* Mv,
                    double sigma, const double* Xi, double* Ti, cudaStream_t st) {
  constexpr int kL = KB <= 4 ? 8 : 4;
  if (spmv_version() == 1)
    spmm_op_k<KB><<<div_up(n * 32, 256), 256, 0, st>>>(n, rp, col, Cv, Mv, sigma, Xi, Ti);
  else
    spmm_op_k2<KB, 5, kL><<<div_up(n * kL, 256), 256, 0, st>>>(n, rp, col, Cv, Mv, sigma, Xi, Ti);
}

template <int KB>
void launch_spmm_csr(int64_t n, const int64_t* rp, const int32_t* col, const double* val, const double* Xi, int w,
                     double* Y, int64_t ldy, cudaStream_t st) {
  constexpr int kL = KB <= 4 ? 8 : 4;
  if (spmv_version() == 1)
    spmm_csr_k<KB><<<div_up(n * 32, 256), 256, 0, st>>>(n, rp, col, val, Xi, w, Y, ldy);
  else
    spmm_csr_k2<KB, 5, kL><<<div_up(n * kL, 256), 256, 0, st>>>(n, rp, col, val, Xi, w, Y, ldy);
}

}  // namespace

// part[(b * k + i) * bs + j] = V[i][chunk b] . R[j][chunk b]: the block stages
// its chunk of the bs vectors of R in shared memory ([j][t], conflict-free),
// each warp owns basis vectors i = warp (mod 8), four at a time; every basis
// entry loaded from HBM feeds bs multiply-adds (block CGS projection)
template <int KB>
__global__ void __launch_bounds__(kRedThreads) gemm_t_part(const double* __restrict__ V, int k, int64_t n2,
                                                         const double* __restrict__ R, int bs, int64_t chunk,
                                                         double* __restrict__ part) {
  extern __shared__ double rs[];
  const int64_t e0 = blockIdx.x * chunk;
  const int len = static_cast<int>(min(chunk, n2 - e0));
  for (int j = 0; j < bs; ++j)
    for (int t = threadIdx.x; t < len; t += kRedThreads) rs[j * chunk + t] = R[j * n2 + e0 + t];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kW = kRedThreads / 32, kV = 4;
  for (int i = warp; i < k; i += kV * kW) {
    const double* vp[kV];
#pragma unroll
    for (int q = 0; q < kV; ++q) vp[q] = V + (int64_t)(i + q * kW < k ? i + q * kW : i) * n2 + e0;
    double acc[kV][KB];
#pragma unroll
    for (int q = 0; q < kV; ++q)
#pragma unroll
      for (int j = 0; j < KB; ++j) acc[q][j] = 0.0;
    int t = lane;
    for (; t + 32 < len; t += 64) {
      double a[kV][2];
#pragma unroll
      for (int q = 0; q < kV; ++q) a[q][0] = vp[q][t], a[q][1] = vp[q][t + 32];
#pragma unroll
      for (int j = 0; j < KB; ++j)
        if (j < bs) {
          const double x0 = rs[j * chunk + t], x1 = rs[j * chunk + t + 32];
#pragma unroll
          for (int q = 0; q < kV; ++q) acc[q][j] += a[q][0] * x0 + a[q][1] * x1;
        }
    }
    for (; t < len; t += 32) {
      double a[kV];
#pragma unroll
      for (int q = 0; q < kV; ++q) a[q] = vp[q][t];
#pragma unroll
      for (int j = 0; j < KB; ++j)
        if (j < bs) {
          const double x0 = rs[j * chunk + t];
#pragma unroll
          for (int q = 0; q < kV; ++q) acc[q][j] += a[q] * x0;
        }
    }
#pragma unroll
    for (int q = 0; q < kV; ++q)
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        const double sq = warp_sum(acc[q][j]);
        if (lane == 0 && j < bs && i + q * kW < k) part[((int64_t)blockIdx.x * k + i + q * kW) * bs + j] = sq;
      }
  }
}

// Persistent form of gemm_t_part: block g takes chunks g, g + G, ... (G =
// gridDim.x), keeps its k x bs sums in shared memory (entry (i, j) is owned
// by warp i mod 8, so no races) and writes them once: G partial rows instead
// of one per chunk, so the final reduction reads G (a few hundred) rows with
// coalesced loads. 16 loads in flight per lane (4 vectors x 4 entries).
template <int KB>
__global__ void __launch_bounds__(kRedThreads) gemm_t_pers(const double* __restrict__ V, int k, int64_t n2,
                                                         const double* __restrict__ R, int bs, int chunk, int nchunks,
                                                         double* __restrict__ part) {
  extern __shared__ double smem[];
  double* rs = smem;                    // [j][chunk]
  double* hsum = smem + KB * chunk;     // [i][bs]
  for (int x = threadIdx.x; x < k * bs; x += kRedThreads) hsum[x] = 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kW = kRedThreads / 32, kV = 4;
  for (int b = blockIdx.x; b < nchunks; b += gridDim.x) {
    const int64_t e0 = (int64_t)b * chunk;
    const int len = static_cast<int>(min((int64_t)chunk, n2 - e0));
    __syncthreads();  // the previous chunk is done with rs
    for (int j = 0; j < bs; ++j)
      for (int t = threadIdx.x; t < len; t += kRedThreads) rs[j * chunk + t] = R[j * n2 + e0 + t];
    __syncthreads();
    for (int i = warp; i < k; i += kV * kW) {
      const double* vp[kV];
#pragma unroll
      for (int q = 0; q < kV; ++q) vp[q] = V + (int64_t)(i + q * kW < k ? i + q * kW : i) * n2 + e0;
      double acc[kV][KB];
#pragma unroll
      for (int q = 0; q < kV; ++q)
#pragma unroll
        for (int j = 0; j < KB; ++j) acc[q][j] = 0.0;
      int t = lane;
      for (; t + 96 < len; t += 128) {
        double a[kV][4];
#pragma unroll
        for (int q = 0; q < kV; ++q)
#pragma unroll
          for (int u = 0; u < 4; ++u) a[q][u] = vp[q][t + 32 * u];
#pragma unroll
        for (int j = 0; j < KB; ++j)
          if (j < bs) {
            const double* xr = rs + j * chunk + t;
            const double x0 = xr[0], x1 = xr[32], x2 = xr[64], x3 = xr[96];
#pragma unroll
            for (int q = 0; q < kV; ++q) acc[q][j] += (a[q][0] * x0 + a[q][1] * x1) + (a[q][2] * x2 + a[q][3] * x3);
          }
      }
      for (; t < len; t += 32) {
        double a[kV];
#pragma unroll
        for (int q = 0; q < kV; ++q) a[q] = vp[q][t];
#pragma unroll
        for (int j = 0; j < KB; ++j)
          if (j < bs) {
            const double x0 = rs[j * chunk + t];
#pragma unroll
            for (int q = 0; q < kV; ++q) acc[q][j] += a[q] * x0;
          }
      }
#pragma unroll
      for (int q = 0; q < kV; ++q)
#pragma unroll
        for (int j = 0; j < KB; ++j) {
          const double sq = warp_sum(acc[q][j]);
          if (lane == 0 && j < bs && i + q * kW < k) hsum[(i + q * kW) * bs + j] += sq;
        }
    }
  }
  __syncthreads();
  for (int x = threadIdx.x; x < k * bs; x += kRedThreads) part[(int64_t)blockIdx.x * k * bs + x] = hsum[x];
}

// H[i + j ldh] = sum_g part[g * k bs + i bs + j]: 32 consecutive entries per
// block, its 8 warps take every 8th partial row (coalesced 256-byte loads),
// combined in warp order (deterministic)
__global__ void __launch_bounds__(256) reduce_rows_k(const double* __restrict__ part, int g, int kb, int bs,
                                                     double* __restrict__ H, int ldh) {
  __shared__ double red[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (x < kb)
    for (int r = warp; r < g; r += 8) s += part[(int64_t)r * kb + x];
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && x < kb) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][lane];
    H[x / bs + (int64_t)(x % bs) * ldh] = t;
  }
}

// H[i + j ldh] = sum_b part[(b * k + i) * bs + j] (fixed order), one warp per entry
__global__ void reduce_parts_blk(const double* __restrict__ part, int nb, int k, int bs, double* __restrict__ H,
                                 int ldh) {
  const int i = blockIdx.x, j = blockIdx.y, lane = threadIdx.x;
  double s = 0.0;
  for (int b = lane; b < nb; b += 32) s += part[((int64_t)b * k + i) * bs + j];
  s = warp_sum(s);
  if (lane == 0) H[i + (int64_t)j * ldh] = s;
}

// R[:, j] -= V[:, 0:k] H[0:k, j], j < bs: one pass over V (each entry feeds bs
// multiply-adds), H staged in shared memory
template <int KB>
__global__ void gemm_n_k(const double* __restrict__ V, int k, int64_t n2, const double* __restrict__ H, int ldh,
                         int bs, double* __restrict__ R) {
  extern __shared__ double hs[];  // [i][KB]
  for (int idx = threadIdx.x; idx < k * KB; idx += blockDim.x) {
    const int i = idx / KB, j = idx % KB;
    hs[idx] = j < bs ? H[i + (int64_t)j * ldh] : 0.0;
  }
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n2; e += (int64_t)gridDim.x * blockDim.x) {
    double s[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j) s[j] = 0.0;
    int i = 0;
    for (; i + 7 < k; i += 8) {  // 8 loads in flight per thread
      double a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = V[(int64_t)(i + u) * n2 + e];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int j = 0; j < KB; ++j) s[j] += a[u] * hs[(i + u) * KB + j];
    }
    for (; i < k; ++i) {
      const double a = V[(int64_t)i * n2 + e];
#pragma unroll
      for (int j = 0; j < KB; ++j) s[j] += a * hs[i * KB + j];
    }
#pragma unroll
    for (int j = 0; j < KB; ++j)
      if (j < bs) R[j * n2 + e] -= s[j];
  }
}

// out[i] = sum_b part[i * nb + b], one warp per output (fixed order)
__global__ void sum_rows(const double* __restrict__ part, int nb, double* __restrict__ out) {
  double s = 0.0;
  for (int b = threadIdx.x; b < nb; b += 32) s += part[(int64_t)blockIdx.x * nb + b];
  s = warp_sum(s);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}


// ---------------------------------------------------------------------------
// From host arrays: the pattern and K, C, M are uploaded once (pageable
// copies) into a temporary device pencil and the device constructor forms
// varsigma, the scaled C / M, Q(s) and the 1-norms there (the same rounding as
// the host formulas: the resident-pencil test checks the two paths bitwise).
std::unique_ptr<DevicePencil> OperatorEngine::upload_pencil(int64_t n, const int64_t* rowptr, const int32_t* col,
                                                            const double* K, const double* C, const double* M) {
  SetupTrace tr("OperatorEngine(host)");
  auto dp = std::make_unique<DevicePencil>();
  dp->n = n;
  dp->nnz = rowptr[n];
  RQB_CUDA(cudaGetDevice(&dp->device));
  const int64_t nnz = dp->nnz;
  dp->d_rowptr.alloc(sizeof(int64_t) * (n + 1));
  dp->d_col.alloc(sizeof(int32_t) * std::max<int64_t>(nnz, 1));
  dp->d_val.alloc(sizeof(double) * std::max<int64_t>(3 * nnz, 1));
  upload_host_sync(dp->d_rowptr.p, rowptr, sizeof(int64_t) * (n + 1), nullptr);
  upload_host_sync(dp->d_col.p, col, sizeof(int32_t) * nnz, nullptr);
  double* v = dp->d_val.as<double>();
  upload_host_sync(v, K, sizeof(double) * nnz, nullptr);
  upload_host_sync(v + nnz, C, sizeof(double) * nnz, nullptr);
  upload_host_sync(v + 2 * nnz, M, sizeof(double) * nnz, nullptr);
  tr.mark("uploads");
  return dp;
}

OperatorEngine::OperatorEngine(int64_t n_, const int64_t* rowptr, const int32_t* col, const double* K,
                               const double* C, const double* M, const Symbolic& s, double sigma_, bool scaling,
                               double* norms1)
    : OperatorEngine(*upload_pencil(n_, rowptr, col, K, C, M), rowptr, col, s, sigma_, scaling, norms1) {}

namespace {

// max |K|, max |M| (non-negative doubles order like their bit patterns:
// exact and order independent)
__global__ void maxabs2_k(int64_t nnz, const double* K, const double* M, unsigned long long* out) {
  double a = 0.0, b = 0.0;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    a = fmax(a, fabs(K[k]));
    b = fmax(b, fabs(M[k]));
  }
  for (int o = 16; o > 0; o >>= 1) {
    a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(a)));
    atomicMax(out + 1, static_cast<unsigned long long>(__double_as_longlong(b)));
  }
}

// Cs = v C, Ms = v2 M (when scaling), Q = K + s C + s^2 M: the host
// constructor's expressions, each product / sum rounded separately
__global__ void pencil_scale_k(int64_t nnz, const double* K, const double* C, const double* M,
                               int scaling, double v, double v2, double s, double* Cs, double* Ms,
                               double* Q) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double c = C[k], m = M[k];
    Cs[k] = scaling ? __dmul_rn(v, c) : c;
    Ms[k] = scaling ? __dmul_rn(v2, m) : m;
    Q[k] = __dadd_rn(__dadd_rn(K[k], __dmul_rn(s, c)), __dmul_rn(__dmul_rn(s, s), m));
  }
}

// 1-norm of f A for the three (A, f) = (K, 1), (C, v), (M, v*v): column sums
// of a symmetric matrix = row sums, each row summed sequentially in column
// order — the same sequence the host's column accumulation adds
__global__ void norm1_sym_k(int64_t n, const int64_t* rowptr, const double* K, const double* C,
                            const double* M, double v, unsigned long long* out) {
  double a[3] = {0.0, 0.0, 0.0};
  const double vv = __dmul_rn(v, v);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double sk = 0.0, sc = 0.0, sm = 0.0;
    for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) {
      sk = __dadd_rn(sk, fabs(K[k]));
      sc = __dadd_rn(sc, fabs(__dmul_rn(v, C[k])));
      sm = __dadd_rn(sm, fabs(__dmul_rn(vv, M[k])));
    }
    a[0] = fmax(a[0], sk);
    a[1] = fmax(a[1], sc);
    a[2] = fmax(a[2], sm);
  }
  for (int i = 0; i < 3; ++i) {
    double x = a[i];
    for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out + i, static_cast<unsigned long long>(__double_as_longlong(x)));
  }
}

}  // namespace

OperatorEngine::OperatorEngine(const DevicePencil& dp, const int64_t* rowptr_h, const int32_t* col_h,
                               const Symbolic& s, double sigma_, bool scaling, double* norms1)
    : n(dp.n) {
  nnz = dp.nnz;
  int dev = 0;
  RQB_CUDA(cudaGetDevice(&dev));
  if (dev != dp.device) fail(errc::config, "device pencil lives on another CUDA device");
  if (rowptr_h[n] != nnz) fail(errc::config, "device pencil / host pattern mismatch");
  SetupTrace tr("OperatorEngine(device)");
  fac = std::make_unique<FactorEngine>(s, n, rowptr_h, col_h, nullptr, dp.d_rowptr.as<int64_t>(),
                                       dp.d_col.as<int32_t>());
  tr.mark("FactorEngine");
  stream = fac->stream;
  d_rowptr.alloc(sizeof(int64_t) * (n + 1));
  d_col.alloc(sizeof(int32_t) * nnz);
  RQB_CUDA(cudaMemcpyAsync(d_rowptr.p, dp.d_rowptr.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, stream));
  RQB_CUDA(cudaMemcpyAsync(d_col.p, dp.d_col.p, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice, stream));
  d_K.alloc(sizeof(double) * nnz);
  RQB_CUDA(cudaMemcpyAsync(d_K.p, dp.K(), sizeof(double) * nnz, cudaMemcpyDeviceToDevice, stream));
  d_C.alloc(sizeof(double) * nnz);
  d_M.alloc(sizeof(double) * nnz);
  d_Q.alloc(sizeof(double) * nnz);
  DeviceBuffer d_red;
  d_red.alloc(sizeof(unsigned long long) * 8);
  unsigned long long* red = d_red.as<unsigned long long>();
  unsigned long long h_red[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  RQB_CUDA(cudaMemsetAsync(red, 0, sizeof(unsigned long long) * 8, stream));
  const int grid = 148 * 8;
  varsigma = 1.0;
  if (scaling) {
    maxabs2_k<<<grid, 256, 0, stream>>>(nnz, dp.K(), dp.M(), red);
    RQB_CUDA(cudaGetLastError());
    RQB_CUDA(cudaMemcpyAsync(h_red, red, sizeof(unsigned long long) * 2, cudaMemcpyDeviceToHost, stream));
    RQB_CUDA(cudaStreamSynchronize(stream));
    double mk, mm;
    std::memcpy(&mk, &h_red[0], sizeof(double));
    std::memcpy(&mm, &h_red[1], sizeof(double));
    if (!(mm > 0)) fail(errc::domain, "scale_pencil: zero M norm");
    varsigma = std::sqrt(mk / mm);
  }
  sigma = sigma_ / varsigma;
  const double v = varsigma, v2 = varsigma * varsigma;
  pencil_scale_k<<<grid, 256, 0, stream>>>(nnz, dp.K(), dp.C(), dp.M(), scaling ? 1 : 0, v, v2, sigma_,
                                           d_C.as<double>(), d_M.as<double>(), d_Q.as<double>());
  RQB_CUDA(cudaGetLastError());
  norm1_sym_k<<<div_up(n, 256), 256, 0, stream>>>(n, d_rowptr.as<int64_t>(), dp.K(), dp.C(), dp.M(), v,
                                                  red + 2);
  RQB_CUDA(cudaGetLastError());
  RQB_CUDA(cudaMemcpyAsync(h_red + 2, red + 2, sizeof(unsigned long long) * 3, cudaMemcpyDeviceToHost, stream));
  fac->set_values_device(d_Q.as<double>());
  RQB_CUDA(cudaStreamSynchronize(stream));
  if (norms1)
    for (int i = 0; i < 3; ++i) std::memcpy(&norms1[i], &h_red[2 + i], sizeof(double));
  tr.mark("scale+Q+norms");
  init_workspaces();
}

void OperatorEngine::init_workspaces() {
  SetupTrace tr("init_workspaces");
  d_w.alloc(sizeof(double) * 2 * n);
  d_t.alloc(sizeof(double) * 2 * n);
  nparts = kRedBlocks;
  // CGS projection: chunks of 256..4096 entries, about 4 blocks per SM when n is large
  gemv_t_chunk = std::min<int64_t>(4096, std::max<int64_t>(256, ((2 * n + kRedBlocks - 1) / kRedBlocks + 255) / 256 * 256));
  gemv_t_blocks = static_cast<int>((2 * n + gemv_t_chunk - 1) / gemv_t_chunk);
  d_part.alloc(sizeof(double) * std::max(kRedBlocks, gemv_t_blocks) * 512);
  d_scal.alloc(sizeof(double) * 64);
  RQB_CUDA(cudaStreamSynchronize(stream));
  tr.mark("alloc");
  fac->factor();
  tr.mark("factor");
}

OperatorEngine::~OperatorEngine() {
}

void OperatorEngine::spmv(int which, const double* x, double* y) {
  const double* val = which == 0 ? d_K.as<double>()
                      : which == 1 ? d_C.as<double>()
                      : which == 2 ? d_M.as<double>()
                                   : d_Q.as<double>();
  launch_spmv_csr(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(), val, x, y, stream);
  ++launches;
}

void OperatorEngine::apply(const double* v, double* r) {
  double* t = d_t.as<double>();
  launch_spmv_op(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(), d_C.as<double>(), d_M.as<double>(), sigma, v, v + n,
                 t, stream);
  ++launches;
  // r_u = -Q(s)^{-1} t ; r_l = s r_u + v_u (fused in the backward sweep)
  rqb_solve_enqueue(*fac, t, r, -1.0, v, sigma, r + n);
  launches += fac->launches_solve;
}

void OperatorEngine::bvec(const double* r, double* w) {
  RQB_CUDA(cudaMemcpyAsync(w, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream));
  spmv(2, r + n, w + n);
}

void OperatorEngine::gemv_t(const double* V, int k, const double* w, double* h) {
  if (k <= 0) return;
  if (k > 512) fail(errc::config, "Krylov dimension above 512");
  gemv_t_part<<<gemv_t_blocks, kRedThreads, sizeof(double) * gemv_t_chunk, stream>>>(
      V, k, 2 * n, w, w + n, n, gemv_t_chunk, d_part.as<double>());
  reduce_parts<<<k, 32, 0, stream>>>(d_part.as<double>(), gemv_t_blocks, k, h, nullptr);
  launches += 2;
}

void OperatorEngine::gemv_n(const double* V, int k, const double* h, double* r, double* h_acc) {
  if (k <= 0) return;
  gemv_n_k<<<std::min(div_up(2 * n, 256), 148 * 8), 256, sizeof(double) * k, stream>>>(V, k, 2 * n, 2 * n,
                                                                                     h, r);
  ++launches;
  (void)h_acc;
}

void OperatorEngine::apply_block(const double* V, int bs, double* R) {
  if (bs <= 0) return;
  if (bs > 8) fail(errc::config, "block size above 8");
  if (d_tb.bytes < sizeof(double) * n * 8 * 3) d_tb.alloc(sizeof(double) * n * 8 * 3);
  double* Xi = d_tb.as<double>();          // 2n x KB interleaved block
  double* Ti = Xi + 2 * n * 8;             // n x KB interleaved SpMM output
  const int64_t n2 = 2 * n;
  const int grid = std::min(div_up(n2, 256), 148 * 8);
  const int kb = bs <= 4 ? 4 : 8;
  if (kb == 4) {
    interleave_k<4><<<grid, 256, 0, stream>>>(V, n2, n2, bs, Xi);
    launch_spmm_op<4>(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(), d_C.as<double>(), d_M.as<double>(), sigma, Xi,
                        Ti, stream);
  } else {
    interleave_k<8><<<grid, 256, 0, stream>>>(V, n2, n2, bs, Xi);
    launch_spmm_op<8>(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(), d_C.as<double>(), d_M.as<double>(), sigma, Xi,
                        Ti, stream);
  }
  launches += 2;
  // R_u = -Q(s)^{-1} T ; R_l = s R_u + V_u (fused in the backward sweep), bs vectors per pass
  rqb_msolve_enqueue(*fac, Ti, 1, bs, R, n2, -1.0, V, n2, sigma, R + n, kb);
  launches += fac->launches_solve;
}

void OperatorEngine::mspmv_block(const double* R, int w, double* Wl) {
  if (w <= 0) return;
  if (d_tb.bytes < sizeof(double) * n * 8 * 3) d_tb.alloc(sizeof(double) * n * 8 * 3);
  double* Xi = d_tb.as<double>();
  const int64_t n2 = 2 * n;
  const int grid = std::min(div_up(n, 256), 148 * 8);
  if (w <= 4) {
    interleave_k<4><<<grid, 256, 0, stream>>>(R + n, n2, n, w, Xi);
    launch_spmm_csr<4>(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(), d_M.as<double>(), Xi, w, Wl, n, stream);
  } else {
    interleave_k<8><<<grid, 256, 0, stream>>>(R + n, n2, n, w, Xi);
    launch_spmm_csr<8>(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(), d_M.as<double>(), Xi, w, Wl, n, stream);
  }
  launches += 2;
}

void OperatorEngine::gemv_n_len(const double* V, int k, int64_t ldv, int64_t len, const double* h, double* r) {
  if (k <= 0) return;
  gemv_n_k<<<std::min(div_up(len, 256), 148 * 8), 256, sizeof(double) * k, stream>>>(V, k, ldv, len, h, r);
  ++launches;
}

void OperatorEngine::prepare_block(int kmax, int bs) {
  rqb_msolve_prepare(*fac);
  if (d_tb.bytes < sizeof(double) * n * 8 * 3) d_tb.alloc(sizeof(double) * n * 8 * 3);
  const int64_t nb = (2 * n + 511) / 512;
  const size_t need = sizeof(double) * static_cast<size_t>(nb) * kmax * bs;
  if (d_bpart.bytes < need) d_bpart.alloc(need);
}

void OperatorEngine::gemm_t(const double* V, int k, const double* R, int bs, double* H, int ldh) {
  if (k <= 0 || bs <= 0) return;
  constexpr int64_t kChunk = 512;
  const int64_t n2 = 2 * n;
  const int nb = static_cast<int>((n2 + kChunk - 1) / kChunk);
  const size_t need = sizeof(double) * static_cast<size_t>(nb) * k * bs;
  if (d_bpart.bytes < need) d_bpart.alloc(need);
  // (width 8 keeps the per-chunk form: its persistent variant needs 140
  // registers, one block per SM, and measured slower: 0.61 -> 0.72 ms at k = 160)
  static const bool pers = !std::getenv("RQB_GEMMT") || std::atoi(std::getenv("RQB_GEMMT")) != 1;
  if (pers && bs <= 4) {
    // persistent: one wave of resident blocks (smem: the R chunk + the k x bs sums)
    const size_t sm = sizeof(double) * (static_cast<size_t>(kChunk) * 4 + static_cast<size_t>(k) * bs);
    auto kern = gemm_t_pers<4>;
    smem_at_least(kern, sm);
    int occ = 1;
    RQB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kRedThreads, sm));
    const int g = std::min(nb, 148 * std::max(1, occ));
    kern<<<g, kRedThreads, sm, stream>>>(V, k, n2, R, bs, static_cast<int>(kChunk), nb, d_bpart.as<double>());
    reduce_rows_k<<<div_up(static_cast<int64_t>(k) * bs, 32), 256, 0, stream>>>(d_bpart.as<double>(), g, k * bs, bs,
                                                                                H, ldh);
    launches += 2;
    return;
  }
  const size_t sm = sizeof(double) * kChunk * bs;
  if (bs <= 4)
    gemm_t_part<4><<<nb, kRedThreads, sm, stream>>>(V, k, n2, R, bs, kChunk, d_bpart.as<double>());
  else
    gemm_t_part<8><<<nb, kRedThreads, sm, stream>>>(V, k, n2, R, bs, kChunk, d_bpart.as<double>());
  reduce_parts_blk<<<dim3(k, bs), 32, 0, stream>>>(d_bpart.as<double>(), nb, k, bs, H, ldh);
  launches += 2;
}

void OperatorEngine::gemm_n(const double* V, int k, const double* H, int ldh, double* R, int bs) {
  if (k <= 0 || bs <= 0) return;
  const int64_t n2 = 2 * n;
  const int grid = std::min(div_up(n2, 256), 148 * 8);
  if (bs <= 4)
    gemm_n_k<4><<<grid, 256, sizeof(double) * k * 4, stream>>>(V, k, n2, H, ldh, bs, R);
  else
    gemm_n_k<8><<<grid, 256, sizeof(double) * k * 8, stream>>>(V, k, n2, H, ldh, bs, R);
  ++launches;
}

void OperatorEngine::dot2n(const double* x, const double* y, double* out) {
  dot_part<<<kRedBlocks, kRedThreads, 0, stream>>>(x, x + n, y, y + n, n, 2 * n, d_part.as<double>());
  sum_parts<<<1, 32, 0, stream>>>(d_part.as<double>(), kRedBlocks, out);
  launches += 2;
}

// w = B r from one M-product (t = M r_l), beta = sqrt(r . w), and both
// v = r / beta and B v = w / beta written in one pass
__global__ void normalize_b_k(const double* __restrict__ part, int nb, const double* __restrict__ r,
                              const double* __restrict__ t, int64_t n, double* __restrict__ beta_out,
                              double* __restrict__ v, double* __restrict__ bv) {
  __shared__ double beta_s;
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int b = threadIdx.x; b < nb; b += 32) s += part[b];
    s = warp_sum(s);
    if (threadIdx.x == 0) {
      const double beta = sqrt(fmax(s, 0.0));
      beta_s = beta;
      if (blockIdx.x == 0 && beta_out) *beta_out = beta;
    }
  }
  __syncthreads();
  const double inv = beta_s > 0.0 ? 1.0 / beta_s : 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 2 * n; e += (int64_t)gridDim.x * blockDim.x) {
    const double re = r[e];
    v[e] = re * inv;
    bv[e] = (e < n ? re : t[e - n]) * inv;
  }
}

void OperatorEngine::bnorm_normalize_b(const double* r, double* beta_out, double* v_next, double* bv_next) {
  double* t = d_t.as<double>();
  spmv(2, r + n, t);  // t = M r_l
  dot_part<<<kRedBlocks, kRedThreads, 0, stream>>>(r, r + n, r, t, n, 2 * n, d_part.as<double>());
  normalize_b_k<<<std::min(div_up(2 * n, 256), 148 * 8), 256, 0, stream>>>(d_part.as<double>(), kRedBlocks, r, t,
                                                                          n, beta_out, v_next, bv_next);
  launches += 2;
}

void OperatorEngine::bnorm_normalize_w(const double* r, const double* wl, double* beta_out, double* v_next,
                                       double* bv_next) {
  dot_part<<<kRedBlocks, kRedThreads, 0, stream>>>(r, r + n, r, wl, n, 2 * n, d_part.as<double>());
  normalize_b_k<<<std::min(div_up(2 * n, 256), 148 * 8), 256, 0, stream>>>(d_part.as<double>(), kRedBlocks, r, wl,
                                                                          n, beta_out, v_next, bv_next);
  launches += 2;
}

void OperatorEngine::bnorm_normalize(const double* r, const double* w, double* beta_out,
                                     double* v_next) {
  dot_part<<<kRedBlocks, kRedThreads, 0, stream>>>(r, r + n, w, w + n, n, 2 * n, d_part.as<double>());
  normalize_k<<<std::min(div_up(2 * n, 256), 148 * 8), 256, 0, stream>>>(
      d_part.as<double>(), kRedBlocks, r, 2 * n, beta_out, v_next);
  launches += 2;
}

void OperatorEngine::combine(const double* V, int k, const double* Q_dev, int ldq, int ncols,
                             double* Vout) {
  if (ncols <= 0 || k <= 0) return;
  // Vout (2n x ncols, column-major) = V (2n x k, basis vectors contiguous) * Q (k x ncols)
  const int64_t n2 = 2 * n;
  vq_gemm(V, n2, n2, k, Q_dev, ldq, ncols, Vout, n2, false, stream);
  ++launches;
}


void OperatorEngine::ritz_residuals(const double* V, int m, const double* Y, int nc, const double* lam,
                                    const int* blk, double* Xrm, double* out) {
  if (nc <= 0) return;
  const int64_t n2 = 2 * n;
  const int ldx = 2 * nc;
  // Xrm (2n x 2nc, row-major) = V (2n x m) Y (m x 2nc)
  vq_gemm(V, n2, n2, m, Y, m, ldx, Xrm, ldx, true, stream);
  if (d_rcand.bytes < sizeof(double) * 2 * nc + sizeof(int) * nc) d_rcand.alloc(sizeof(double) * 2 * nc + sizeof(int) * nc);
  const int nbx = kRedBlocks;
  if (d_rpart.bytes < sizeof(double) * 8 * nc * nbx) d_rpart.alloc(sizeof(double) * 8 * nc * nbx);
  std::vector<char> hbuf(sizeof(double) * 2 * nc + sizeof(int) * nc);
  std::memcpy(hbuf.data(), lam, sizeof(double) * 2 * nc);
  std::memcpy(hbuf.data() + sizeof(double) * 2 * nc, blk, sizeof(int) * nc);
  RQB_CUDA(cudaMemcpyAsync(d_rcand.p, hbuf.data(), hbuf.size(), cudaMemcpyHostToDevice, stream));
  const double* dlam = d_rcand.as<double>();
  const int* dblk = reinterpret_cast<const int*>(dlam + 2 * nc);
  dim3 grid(nbx, (nc + 63) / 64);
  ritz_residual_k<<<grid, kRedThreads, 0, stream>>>(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(), d_K.as<double>(),
                                                   d_C.as<double>(), d_M.as<double>(), Xrm, ldx, nc, dlam, dblk,
                                                   d_rpart.as<double>());
  sum_rows<<<8 * nc, 32, 0, stream>>>(d_rpart.as<double>(), nbx, out);
  launches += 3;
}

void OperatorEngine::residuals_again(const double* Xrm, int nc, const double* lam, double* out) {
  if (nc <= 0) return;
  const int nbx = kRedBlocks;
  RQB_CUDA(cudaMemcpyAsync(d_rcand.p, lam, sizeof(double) * 2 * nc, cudaMemcpyHostToDevice, stream));
  const double* dlam = d_rcand.as<double>();
  const int* dblk = reinterpret_cast<const int*>(dlam + 2 * nc);
  dim3 grid(nbx, (nc + 63) / 64);
  ritz_residual_k<<<grid, kRedThreads, 0, stream>>>(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(), d_K.as<double>(),
                                                   d_C.as<double>(), d_M.as<double>(), Xrm, 2 * nc, nc, dlam, dblk,
                                                   d_rpart.as<double>());
  sum_rows<<<8 * nc, 32, 0, stream>>>(d_rpart.as<double>(), nbx, out);
  launches += 2;
}

void OperatorEngine::ritz_extract(const double* Xrm, int nc, int c, int part_im, double* out) {
  const int* dblk = reinterpret_cast<const int*>(d_rcand.as<double>() + 2 * nc);
  ritz_extract_k<<<std::min(div_up(n, 256), kRedBlocks), 256, 0, stream>>>(Xrm, 2 * nc, n, dblk, c, part_im, out);
  ++launches;
}


double OperatorEngine::time_op(int what, int iters, int param) {
  const bool flush_l2 = (what & 0x100) != 0;
  what &= 0xff;
  const int64_t n2 = 2 * n;
  const int k = std::max(1, std::min(param, 511));
  DeviceBuffer a, b, V, h;
  a.alloc(sizeof(double) * n2);
  b.alloc(sizeof(double) * n2);
  DeviceBuffer Q, X;
  std::vector<double> lamh;
  std::vector<int> blkh;
  if (what == 7 || what == 8) {  // restart DGEMM 2n x k x k / batched residual of k candidates
    V.alloc(sizeof(double) * k * n2);
    Q.alloc(sizeof(double) * k * k);
    X.alloc(sizeof(double) * k * n2);
    RQB_CUDA(cudaMemsetAsync(V.p, 0, V.bytes, stream));
    RQB_CUDA(cudaMemsetAsync(Q.p, 0, Q.bytes, stream));
    for (int c = 0; c < k; ++c) lamh.push_back(0.1), lamh.push_back(0.2), blkh.push_back(c & 1);
    h.alloc(sizeof(double) * 8 * k);
  }
  DeviceBuffer Vb, Rb;
  const int kb = std::max(1, std::min(8, param >> 16));  // what 11 / 12: block width in the high bits
  if (what == 11 || what == 12) {  // block CGS projection / update over k = param & 0xffff basis vectors
    V.alloc(sizeof(double) * (param & 0xffff) * n2);
    Rb.alloc(sizeof(double) * n2 * 8);
    h.alloc(sizeof(double) * (param & 0xffff) * 8);
    RQB_CUDA(cudaMemsetAsync(V.p, 0, V.bytes, stream));
    RQB_CUDA(cudaMemsetAsync(Rb.p, 0, Rb.bytes, stream));
    RQB_CUDA(cudaMemsetAsync(h.p, 0, h.bytes, stream));
    prepare_block((param & 0xffff) + 8, 8);
  }
  if (what == 9 || what == 10 || what == 13 || what == 14) {  // block apply / multi-RHS solve / block SpMMs
    Vb.alloc(sizeof(double) * n2 * 8);
    Rb.alloc(sizeof(double) * n2 * 8);
    RQB_CUDA(cudaMemsetAsync(Vb.p, 0, Vb.bytes, stream));
    prepare_block(8, 8);
  }
  if (what == 3 || what == 4) {
    V.alloc(sizeof(double) * (k + 1) * n2);
    h.alloc(sizeof(double) * (k + 1));
    RQB_CUDA(cudaMemsetAsync(V.p, 0, V.bytes, stream));
    RQB_CUDA(cudaMemsetAsync(h.p, 0, h.bytes, stream));
  }
  RQB_CUDA(cudaMemsetAsync(a.p, 0, a.bytes, stream));
  auto run = [&]() {
    switch (what) {
      case 0: apply(a.as<double>(), b.as<double>()); break;
      case 1: fac->solve_device(a.as<double>(), b.as<double>(), 1.0); break;
      case 2:
        launch_spmv_op(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(), d_C.as<double>(), d_M.as<double>(), sigma,
                       a.as<double>(), a.as<double>() + n, b.as<double>(), stream);
        break;
      case 13:  // block SpMM of the operator (C, M) on an interleaved block of k (4 or 8) vectors
        if (k <= 4)
          launch_spmm_op<4>(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(), d_C.as<double>(), d_M.as<double>(), sigma,
                            Vb.as<double>(), Rb.as<double>(), stream);
        else
          launch_spmm_op<8>(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(), d_C.as<double>(), d_M.as<double>(), sigma,
                            Vb.as<double>(), Rb.as<double>(), stream);
        break;
      case 14:  // block M-SpMM (intra-block CGS tracking) on an interleaved block of k vectors
        if (k <= 4)
          launch_spmm_csr<4>(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(), d_M.as<double>(), Vb.as<double>(), k,
                             Rb.as<double>(), n, stream);
        else
          launch_spmm_csr<8>(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(), d_M.as<double>(), Vb.as<double>(), k,
                             Rb.as<double>(), n, stream);
        break;
      case 3: gemv_t(V.as<double>(), k, a.as<double>(), h.as<double>()); break;
      case 4: gemv_n(V.as<double>(), k, h.as<double>(), a.as<double>(), nullptr); break;
      case 5: RQB_CUDA(cudaGraphLaunch(fac->graph_factor_exec, stream)); break;
      case 6: spmv(2, a.as<double>(), b.as<double>()); break;
      case 7: combine(V.as<double>(), k, Q.as<double>(), k, k, X.as<double>()); break;
      case 8: ritz_residuals(V.as<double>(), k, Q.as<double>(), k / 2, lamh.data(), blkh.data(), X.as<double>(), h.as<double>()); break;
      case 11: gemm_t(V.as<double>(), param & 0xffff, Rb.as<double>(), kb, h.as<double>(), param & 0xffff); break;
      case 12: gemm_n(V.as<double>(), param & 0xffff, h.as<double>(), param & 0xffff, Rb.as<double>(), kb); break;
      case 9: apply_block(Vb.as<double>(), std::min(k, 8), Rb.as<double>()); break;
      case 10:
        rqb_msolve_enqueue(*fac, Vb.as<double>(), n, std::min(k, 8), Rb.as<double>(), n, 1.0, nullptr, 0, 0.0, nullptr);
        break;
      default: fail(errc::config, "unknown timing target");
    }
  };
  for (int w = 0; w < 3; ++w) run();
  cudaEvent_t e0, e1;
  RQB_CUDA(cudaEventCreate(&e0));
  RQB_CUDA(cudaEventCreate(&e1));
  float total = 0;
  if (flush_l2) {
    // 256 MiB scrub (> 126 MB L2) before every timed call; each call timed alone
    DeviceBuffer scrub;
    scrub.alloc(size_t(256) << 20);
    for (int it = 0; it < iters; ++it) {
      RQB_CUDA(cudaMemsetAsync(scrub.p, it & 0xff, scrub.bytes, stream));
      RQB_CUDA(cudaEventRecord(e0, stream));
      run();
      RQB_CUDA(cudaEventRecord(e1, stream));
      RQB_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      RQB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      total += ms;
    }
  } else {
    RQB_CUDA(cudaEventRecord(e0, stream));
    for (int it = 0; it < iters; ++it) run();
    RQB_CUDA(cudaEventRecord(e1, stream));
    RQB_CUDA(cudaEventSynchronize(e1));
    RQB_CUDA(cudaEventElapsedTime(&total, e0, e1));
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  RQB_CUDA(cudaGetLastError());
  return total / iters;
}

// ---------------------------------------------------------------------------
// Generalized Hermitian-definite path: A, B on one pattern,
// factor of A - s B, operator S = (A - s B)^{-1} B on n-vectors.
namespace {

// q = A - s B on the shared pattern (each product and sum rounded separately)
__global__ void gh_shifted_k(int64_t nnz, const double* A, const double* B, double s, double* Q) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    Q[k] = __dsub_rn(A[k], __dmul_rn(s, B[k]));
}

// r_c = A x_c - lam_c B x_c for one candidate per blockIdx.y, one warp per row;
// partials of ||r||^2 and ||x||^2 per block (fixed order)
__global__ void __launch_bounds__(kRedThreads) gh_residual_k(int64_t n, const int64_t* __restrict__ rowptr,
                                                           const int32_t* __restrict__ col,
                                                           const double* __restrict__ A,
                                                           const double* __restrict__ B,
                                                           const double* __restrict__ X,
                                                           const double* __restrict__ lam,
                                                           double* __restrict__ part) {
  __shared__ double sr[kRedThreads / 32], sx[kRedThreads / 32];
  const int c = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* x = X + (int64_t)c * n;
  const double l = lam[c];
  double accr = 0.0, accx = 0.0;
  for (int64_t row = blockIdx.x * (int64_t)(kRedThreads / 32) + warp; row < n;
       row += (int64_t)gridDim.x * (kRedThreads / 32)) {
    double a = 0.0, b = 0.0;
    for (int64_t k = rowptr[row] + lane; k < rowptr[row + 1]; k += 32) {
      const double xv = x[col[k]];
      a += A[k] * xv;
      b += B[k] * xv;
    }
    a = warp_sum(a);
    b = warp_sum(b);
    const double r = a - l * b;
    accr += r * r;
    accx += x[row] * x[row];
  }
  if (lane == 0) sr[warp] = accr, sx[warp] = accx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) s0 += sr[w], s1 += sx[w];
    part[(int64_t)(2 * c) * gridDim.x + blockIdx.x] = s0;
    part[(int64_t)(2 * c + 1) * gridDim.x + blockIdx.x] = s1;
  }
}

}  // namespace

GhEngine::GhEngine(int64_t n_, const int64_t* rowptr, const int32_t* col, const double* A, const double* B,
                   const Symbolic& s, double shift_)
    : n(n_), shift(shift_) {
  nnz = rowptr[n];
  d_rowptr.alloc(sizeof(int64_t) * (n + 1));
  d_col.alloc(sizeof(int32_t) * std::max<int64_t>(nnz, 1));
  RQB_CUDA(cudaMemcpy(d_rowptr.p, rowptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
  RQB_CUDA(cudaMemcpy(d_col.p, col, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice));
  fac = std::make_unique<FactorEngine>(s, n, rowptr, col, nullptr, d_rowptr.as<int64_t>(), d_col.as<int32_t>());
  stream = fac->stream;
  d_A.upload(A, sizeof(double) * nnz, stream);
  d_B.upload(B, sizeof(double) * nnz, stream);
  DeviceBuffer q;
  q.alloc(sizeof(double) * std::max<int64_t>(nnz, 1));
  gh_shifted_k<<<148 * 8, 256, 0, stream>>>(nnz, d_A.as<double>(), d_B.as<double>(), shift, q.as<double>());
  RQB_CUDA(cudaGetLastError());
  fac->set_values_device(q.as<double>());
  RQB_CUDA(cudaStreamSynchronize(stream));
  d_t.alloc(sizeof(double) * std::max<int64_t>(n, 1));
  gemv_t_chunk = std::min<int64_t>(4096, std::max<int64_t>(256, ((n + kRedBlocks - 1) / kRedBlocks + 255) / 256 * 256));
  gemv_t_blocks = static_cast<int>((n + gemv_t_chunk - 1) / gemv_t_chunk);
  d_part.alloc(sizeof(double) * std::max(kRedBlocks, gemv_t_blocks) * 512);
  fac->factor();
}

void GhEngine::spmv(int which, const double* x, double* y) {
  launch_spmv_csr(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(), which == 0 ? d_A.as<double>() : d_B.as<double>(),
                  x, y, stream);
  ++launches;
}

void GhEngine::apply(const double* v, double* r) {
  spmv(1, v, d_t.as<double>());
  rqb_solve_enqueue(*fac, d_t.as<double>(), r, 1.0, nullptr, 0.0, nullptr);
  launches += fac->launches_solve;
}

void GhEngine::gemv_t(const double* V, int k, const double* w, double* h) {
  if (k <= 0) return;
  if (k > 512) fail(errc::config, "Krylov dimension above 512");
  gemv_t_part<<<gemv_t_blocks, kRedThreads, sizeof(double) * gemv_t_chunk, stream>>>(
      V, k, n, w, w, n, gemv_t_chunk, d_part.as<double>());
  reduce_parts<<<k, 32, 0, stream>>>(d_part.as<double>(), gemv_t_blocks, k, h, nullptr);
  launches += 2;
}

void GhEngine::gemv_n(const double* V, int k, const double* h, double* r) {
  if (k <= 0) return;
  gemv_n_k<<<std::min(div_up(n, 256), 148 * 8), 256, sizeof(double) * k, stream>>>(V, k, n, n, h, r);
  ++launches;
}

void GhEngine::bnorm_normalize(const double* r, double* beta_out, double* v, double* bv) {
  double* t = d_t.as<double>();
  spmv(1, r, t);  // t = B r
  dot_part<<<kRedBlocks, kRedThreads, 0, stream>>>(r, r, t, t, n, n, d_part.as<double>());
  // normalize_k writes v = r / beta; B v = t / beta by a second pass over t
  normalize_k<<<std::min(div_up(n, 256), 148 * 8), 256, 0, stream>>>(d_part.as<double>(), kRedBlocks, r, n,
                                                                    beta_out, v);
  normalize_k<<<std::min(div_up(n, 256), 148 * 8), 256, 0, stream>>>(d_part.as<double>(), kRedBlocks, t, n,
                                                                    nullptr, bv);
  launches += 3;
}

void GhEngine::residuals(const double* X, int nc, const double* lam_host, double* out_host) {
  if (nc <= 0) return;
  const int nbx = kRedBlocks;
  if (d_res.bytes < sizeof(double) * (2 * static_cast<size_t>(nc) * nbx + nc))
    d_res.alloc(sizeof(double) * (2 * static_cast<size_t>(nc) * nbx + nc));
  double* part = d_res.as<double>();
  double* dlam = part + 2 * static_cast<size_t>(nc) * nbx;
  RQB_CUDA(cudaMemcpyAsync(dlam, lam_host, sizeof(double) * nc, cudaMemcpyHostToDevice, stream));
  gh_residual_k<<<dim3(nbx, nc), kRedThreads, 0, stream>>>(n, d_rowptr.as<int64_t>(), d_col.as<int32_t>(),
                                                           d_A.as<double>(), d_B.as<double>(), X, dlam, part);
  std::vector<double> h(2 * static_cast<size_t>(nc) * nbx);
  RQB_CUDA(cudaMemcpyAsync(h.data(), part, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, stream));
  RQB_CUDA(cudaStreamSynchronize(stream));
  launches += 1;
  for (int c = 0; c < 2 * nc; ++c) {
    double sacc = 0.0;
    for (int b = 0; b < nbx; ++b) sacc += h[static_cast<size_t>(c) * nbx + b];
    out_host[c] = sacc;
  }
}

}  // namespace rqb
