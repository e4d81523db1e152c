// SPDX-License-Identifier: Apache-2.0
// Krylov basis products X = V Q on FP64 tensor cores (krylov_schur_restart
// V <- V Q_keep; Ritz vectors V_m y of ritz_extract and the
// explicit residual check).
//
// V is the basis: n2 x k with basis vector j contiguous at V + j * ldv; Q is
// k x c column-major (ldq, any alignment); X is n2 x c, column-major (ldx >= n2:
// the restarted basis) or row-major (ldx >= c: the Ritz-vector batch the
// residual SpMM reads row by row). Tall and skinny: n2 up to 1.2M, k, c <= 512.
//
// One CTA owns a 128-row block of V and 128 columns of X (grid.x = column
// blocks, fastest, so the CTAs sharing a row block run together and the
// second reads hit L2): V is read from HBM once, Q (<= 2 MB) lives in L2.
// The K loop streams 16 basis vectors per stage, three stages in flight by
// cp.async (A: 16-byte copies of 128 contiguous rows per vector; B: 8-byte
// copies, Q's columns need not be 16-byte aligned), and 8 warps (2 along m,
// 4 along n) each run 16 mma.sync.m16n8k4 f64 (DMMA) per k-step on a 64 x 32
// warp tile: 12 shared loads per 16 DMMA. The FP64 path of sm_100a has no
// tcgen05 form (ptxas rejects kind::f64), so warp-level DMMA is the tensor
// path; fragments read shared memory conflict-free (strides = 4 mod 16 doubles).
#include <cuda_runtime.h>

#include <algorithm>

#include "device.cuh"

namespace rqb {

namespace {

constexpr int kBM = 128, kBN = 128, kBK = 16, kStages = 3, kThreads = 256;
constexpr int kAS = kBM + 4;  // As[kk][m] stride (doubles)
constexpr int kBS = kBK + 4;  // Bs[n][kk] stride
constexpr int kStageD = kBK * kAS + kBN * kBS;
constexpr size_t kSmem = sizeof(double) * kStageD * kStages;

__device__ __forceinline__ void mma_f64(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ void cp16(double* smem, const double* gmem, int nvalid) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(8 * nvalid) : "memory");
}

__device__ __forceinline__ void cp8(double* smem, const double* gmem, bool valid) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0) : "memory");
}

template <bool kRowMajor>
__global__ void __launch_bounds__(kThreads, 1)
    vq_gemm_k(const double* __restrict__ V, int64_t ldv, int64_t n2, int k, const double* __restrict__ Q, int ldq,
              int c, double* __restrict__ X, int64_t ldx) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int wm = (warp & 1) * 64, wn = (warp >> 1) * 32;
  const int ncb = (c + kBN - 1) / kBN;  // column blocks fastest: CTAs of one row block run together
  const int64_t r0 = static_cast<int64_t>(blockIdx.x / ncb) * kBM;
  const int c0 = static_cast<int>(blockIdx.x % ncb) * kBN;
  const int nr = static_cast<int>(n2 - r0 < kBM ? n2 - r0 : kBM);
  const int nc = min(kBN, c - c0);
  const int nchunks = (k + kBK - 1) / kBK;
  // a 16-byte A copy needs an even first row and an even leading dimension
  const bool a16 = ((ldv & 1) == 0) && ((reinterpret_cast<uintptr_t>(V) & 15) == 0);

  auto issue = [&](int chunk) {
    double* As = sm + (chunk % kStages) * kStageD;
    double* Bs = As + kBK * kAS;
    const int k0 = chunk * kBK;
    if (a16) {
#pragma unroll
      for (int i = 0; i < kBK * kBM / 2 / kThreads; ++i) {
        const int idx = tid + i * kThreads;
        const int kk = idx / (kBM / 2), m = 2 * (idx % (kBM / 2));
        const int nv = (k0 + kk < k) ? max(0, min(2, nr - m)) : 0;
        cp16(&As[kk * kAS + m], nv ? V + (int64_t)(k0 + kk) * ldv + r0 + m : V, nv);
      }
    } else {
#pragma unroll
      for (int i = 0; i < kBK * kBM / kThreads; ++i) {
        const int idx = tid + i * kThreads;
        const int kk = idx / kBM, m = idx % kBM;
        const bool ok = k0 + kk < k && m < nr;
        cp8(&As[kk * kAS + m], ok ? V + (int64_t)(k0 + kk) * ldv + r0 + m : V, ok);
      }
    }
#pragma unroll
    for (int i = 0; i < kBK * kBN / kThreads; ++i) {
      const int idx = tid + i * kThreads;
      const int col = idx / kBK, kk = idx % kBK;
      const bool ok = col < nc && k0 + kk < k;
      cp8(&Bs[col * kBS + kk], ok ? Q + (int64_t)(c0 + col) * ldq + k0 + kk : Q, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  double acc[4][4][4];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[x][y][e] = 0.0;

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s)
    if (s < nchunks) issue(s);
    else asm volatile("cp.async.commit_group;" ::: "memory");

  for (int ch = 0; ch < nchunks; ++ch) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kStages - 2) : "memory");
    __syncthreads();  // stage ch visible; stage ch-1 fully consumed by every warp
    if (ch + kStages - 1 < nchunks) issue(ch + kStages - 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    const double* As = sm + (ch % kStages) * kStageD;
    const double* Bs = As + kBK * kAS;
#pragma unroll
    for (int ks = 0; ks < kBK / 4; ++ks) {
      const int kr = ks * 4 + tig;
      double af[4][2], bf[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        af[x][0] = As[kr * kAS + wm + x * 16 + gid];
        af[x][1] = As[kr * kAS + wm + x * 16 + gid + 8];
      }
#pragma unroll
      for (int y = 0; y < 4; ++y) bf[y] = Bs[(wn + y * 8 + gid) * kBS + kr];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) mma_f64(acc[x][y], af[x][0], af[x][1], bf[y]);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");

  // epilogue: C fragment (gid | gid + 8, 2 tig | 2 tig + 1) of each m16n8 tile
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = wm + x * 16 + gid + h * 8;
        const int cc = wn + y * 8 + 2 * tig;
        if (r >= nr) continue;
        const int64_t gr = r0 + r;
        if (kRowMajor) {
          double* dst = X + gr * ldx + c0 + cc;
          if (cc + 1 < nc && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
            *reinterpret_cast<double2*>(dst) = make_double2(acc[x][y][2 * h], acc[x][y][2 * h + 1]);
          } else {
            if (cc < nc) dst[0] = acc[x][y][2 * h];
            if (cc + 1 < nc) dst[1] = acc[x][y][2 * h + 1];
          }
        } else {
          if (cc < nc) X[(int64_t)(c0 + cc) * ldx + gr] = acc[x][y][2 * h];
          if (cc + 1 < nc) X[(int64_t)(c0 + cc + 1) * ldx + gr] = acc[x][y][2 * h + 1];
        }
      }
}

}  // namespace

// X = V Q (see the header comment). Enqueued on `stream`; no synchronisation.
void vq_gemm(const double* V, int64_t ldv, int64_t n2, int k, const double* Q, int ldq, int c, double* X,
             int64_t ldx, bool row_major_out, cudaStream_t stream) {
  if (n2 <= 0 || c <= 0) return;
  if (k <= 0) {  // empty product: X = 0
    if (row_major_out)
      RQB_CUDA(cudaMemset2DAsync(X, sizeof(double) * ldx, 0, sizeof(double) * c, n2, stream));
    else
      RQB_CUDA(cudaMemset2DAsync(X, sizeof(double) * ldx, 0, sizeof(double) * n2, c, stream));
    return;
  }
  auto kern = row_major_out ? vq_gemm_k<true> : vq_gemm_k<false>;
  smem_at_least(kern, kSmem);
  const int64_t blocks = (n2 + kBM - 1) / kBM * ((c + kBN - 1) / kBN);
  if (blocks > 2147483647LL) fail(errc::config, "vq_gemm: too many blocks");
  const dim3 grid(static_cast<unsigned>(blocks));
  if (row_major_out)
    vq_gemm_k<true><<<grid, kThreads, kSmem, stream>>>(V, ldv, n2, k, Q, ldq, c, X, ldx);
  else
    vq_gemm_k<false><<<grid, kThreads, kSmem, stream>>>(V, ldv, n2, k, Q, ldq, c, X, ldx);
  RQB_CUDA(cudaGetLastError());
}

}  // namespace rqb
