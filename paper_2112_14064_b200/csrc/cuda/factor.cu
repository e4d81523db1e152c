// SPDX-License-Identifier: Apache-2.0
// Numeric multifrontal LU of Q(sigma) on sm_100a (lu_factorize).
//
// Data layout: every front f owns a dense column-major block of
// the front pool (ld_f x nf_f, ld_f = nf_f rounded up to 4) holding, after
// factorization, L (unit lower, columns 0..npiv-1), U (rows 0..npiv-1) and the
// Schur complement (rows/cols npiv..nf-1) consumed by the parent. The
// reference's per-pivot rank-1 update (`kern::elim_step`, kernels.hpp:33-38,
// kernels.cpp:58-69) becomes:
//   scatter_original   one pass over A's nnz into the zeroed pool (atomic-free:
//                      every CSR entry has a unique front destination)
//   extend_add         gather of the children's Schur blocks into the parent
//                      (each parent entry owned by one thread: atomic-free)
//   front_lu_smem      fronts with nf <= 160: one CTA per front, whole front in
//                      shared memory, warp-shuffle threshold pivot search
//   panel_lu           blocked path, one thread-block cluster per front: the
//                      32-wide candidate panel lives in the cluster's shared
//                      memory (DSMEM), pivot search = CTA argmax + one DSMEM
//                      exchange, explicit inverses of L11/U11 for the TRSMs
//   panel_apply        row swaps outside the panel + U12 = L11^-1 A12 and
//                      L_cb = A_cb U11^-1 (TRSM via the 32x32 inverses)
//   schur_dmma         trailing update A22 -= L21 U12 on FP64 tensor cores
//                      (mma.sync m16n8k4 f64 -> DMMA), 64x64 tiles
// Pivoting: threshold u = 0.1 among fully-summed rows only, prefer the
// diagonal, ties -> lowest row, singular if every candidate < 1e-300
// (SURVEY App. B D2).
#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "device.cuh"

namespace cg = cooperative_groups;

namespace rqb {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    fail(errc::config, std::string("CUDA error: ") + cudaGetErrorString(e) + " in " + what);
  // RQB_CHECK_LAST=1 (debugging): a pending launch error is reported at the
  // first checked call after it
  static const bool check_last = std::getenv("RQB_CHECK_LAST") != nullptr;
  if (check_last) {
    const cudaError_t p = cudaPeekAtLastError();
    if (p != cudaSuccess)
      fail(errc::config, std::string("CUDA error (pending): ") + cudaGetErrorString(p) + " seen at " + what);
  }
}

static double wall_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

SetupTrace::SetupTrace(const char* w) : who(w), on(std::getenv("RQB_SETUP_TRACE") != nullptr), t0(wall_ms()) {}

void SetupTrace::mark(const char* phase) {
  if (!on) return;
  const double t = wall_ms();
  std::fprintf(stderr, "[setup] %s %s %.1f ms\n", who, phase, t - t0);
  t0 = t;
}

DeviceBuffer::~DeviceBuffer() {
  if (p) cudaFree(p);
}

void DeviceBuffer::alloc(size_t nbytes) {
  if (p) cudaFree(p);
  p = nullptr;
  bytes = nbytes;
  if (nbytes) RQB_CUDA(cudaMalloc(&p, nbytes));
}

void DeviceBuffer::upload(const void* src, size_t nbytes, cudaStream_t s) {
  if (nbytes > bytes) alloc(nbytes);
  if (nbytes) RQB_CUDA(cudaMemcpyAsync(p, src, nbytes, cudaMemcpyHostToDevice, s));
}

// ---------------------------------------------------------------------------
__global__ void scatter_original(const double* __restrict__ aval, const int64_t* __restrict__ dst,
                                 int64_t nnz, double* __restrict__ pool) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x)
    pool[dst[i]] = aval[i];
}

// grid: (ceil(maxnf/8), nfronts) block (32, 8)
__global__ void extend_add(const FrontDev* __restrict__ fronts, const int32_t* __restrict__ list,
                           const int32_t* __restrict__ inv, double* __restrict__ pool) {
  const FrontDev F = fronts[list[blockIdx.y]];
  const int c = blockIdx.x * 8 + threadIdx.y;
  if (c >= F.nf) return;
  const int32_t* inv0 = inv + F.inv_off;
  const int32_t* inv1 = inv0 + F.nf;
  const int ic0 = inv0[c];
  const int ic1 = F.nchild > 1 ? inv1[c] : -1;
  if (ic0 < 0 && ic1 < 0) return;
  const FrontDev C0 = fronts[F.child0];
  const double* c0col = pool + C0.off + (int64_t)ic0 * C0.ld;
  const double* c1col = nullptr;
  if (ic1 >= 0) {
    const FrontDev C1 = fronts[F.child1];
    c1col = pool + C1.off + (int64_t)ic1 * C1.ld;
  }
  double* col = pool + F.off + (int64_t)c * F.ld;
  for (int r = threadIdx.x; r < F.nf; r += 32) {
    double acc = 0.0;
    bool any = false;
    if (ic0 >= 0) {
      const int ir = inv0[r];
      if (ir >= 0) acc += c0col[ir], any = true;
    }
    if (ic1 >= 0) {
      const int ir = inv1[r];
      if (ir >= 0) acc += c1col[ir], any = true;
    }
    if (any) col[r] += acc;
  }
}

// ---------------------------------------------------------------------------
// Whole-front LU in shared memory, one CTA per front.
template <int NT>
__global__ void __launch_bounds__(NT) front_lu_smem(const FrontDev* __restrict__ fronts,
                                                   const int32_t* __restrict__ list,
                                                   double* __restrict__ pool,
                                                   int32_t* __restrict__ ipiv,
                                                   int* __restrict__ flags) {
  extern __shared__ double sm[];
  __shared__ double lcol[kSmallNf];
  __shared__ int piv_s;
  const FrontDev F = fronts[list[blockIdx.x]];
  const int nf = F.nf, np = F.npiv;
  if (np == 0) return;
  const int lds = nf;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  double* g = pool + F.off;
  for (int c = warp; c < nf; c += NW)
    for (int r = lane; r < nf; r += 32) sm[r + c * lds] = g[r + (int64_t)c * F.ld];
  for (int k = 0; k < np; ++k) {
    __syncthreads();
    if (warp == 0) {
      double best = -1.0;
      int bi = k;
      for (int i = k + lane; i < np; i += 32) {
        const double v = fabs(sm[i + k * lds]);
        if (v > best) best = v, bi = i;
      }
      warp_argmax(best, bi);
      if (lane == 0) {
        const double diag = fabs(sm[k + k * lds]);
        int p = diag >= kPivThreshold * best ? k : bi;
        if (!(best >= kSingularTiny)) {
          atomicOr(&flags[0], 1);
          p = k;
        }
        if (p != k) atomicAdd(&flags[1], 1);
        piv_s = p;
        ipiv[F.start + k] = p;
      }
    }
    __syncthreads();
    const int p = piv_s;
    if (p != k)
      for (int c = tid; c < nf; c += NT) {
        const double t = sm[k + c * lds];
        sm[k + c * lds] = sm[p + c * lds];
        sm[p + c * lds] = t;
      }
    __syncthreads();
    const double akk = sm[k + k * lds];
    for (int i = k + 1 + tid; i < nf; i += NT) {
      const double l = sm[i + k * lds] / akk;
      sm[i + k * lds] = l;
      lcol[i] = l;
    }
    __syncthreads();
    for (int c = k + 1 + warp; c < nf; c += NW) {
      const double u = sm[k + c * lds];
      if (u != 0.0)
        for (int r = k + 1 + lane; r < nf; r += 32) sm[r + c * lds] -= lcol[r] * u;
    }
  }
  __syncthreads();
  for (int c = warp; c < nf; c += NW)
    for (int r = lane; r < nf; r += 32) g[r + (int64_t)c * F.ld] = sm[r + c * lds];
}

// ---------------------------------------------------------------------------
// Panel LU of candidate rows [k, npiv) x columns [k, k+w), one cluster per front.
struct PanelSlot {
  double val;
  double diag;
  int row;
  int pad;
};

template <int NT>
__global__ void __launch_bounds__(NT) panel_lu(const FrontDev* __restrict__ fronts,
                                              const int32_t* __restrict__ list, int k,
                                              double* __restrict__ pool,
                                              int32_t* __restrict__ ipiv,
                                              double* __restrict__ scratch,
                                              int* __restrict__ flags) {
  extern __shared__ double pan[];
  __shared__ PanelSlot slot;
  __shared__ double urow[kNB], tmprow[kNB];
  __shared__ double wv[NT / 32];
  __shared__ int wi[NT / 32];
  __shared__ int piv_s;
  __shared__ double T[kNB * kNB];
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const FrontDev F = fronts[list[blockIdx.x / cs]];
  const int np = F.npiv;
  const int w = min(kNB, np - k);
  const int R = np - k;
  const int chunk = (R + cs - 1) / cs;
  const int cpad = chunk | 1;
  const int r0 = rank * chunk;
  const int nloc = max(0, min(R, r0 + chunk) - r0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* g = pool + F.off;
  // load my rows of the panel
  for (int c = warp; c < w; c += NT / 32)
    for (int i = lane; i < nloc; i += 32) pan[i + c * cpad] = g[(k + r0 + i) + (int64_t)(k + c) * F.ld];
  __syncthreads();
  for (int j = 0; j < w; ++j) {
    // local argmax over relative rows >= j
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int i = max(0, j - r0) + tid; i < nloc; i += NT) {
      const double v = fabs(pan[i + j * cpad]);
      if (v > best) best = v, bi = r0 + i;
    }
    warp_argmax(best, bi);
    if (lane == 0) wv[warp] = best, wi[warp] = bi;
    __syncthreads();
    if (tid == 0) {
      for (int q = 1; q < NT / 32; ++q)
        if (wv[q] > best || (wv[q] == best && wi[q] < bi)) best = wv[q], bi = wi[q];
      slot.val = best;
      slot.row = bi;
      slot.diag = (j >= r0 && j < r0 + nloc) ? fabs(pan[(j - r0) + j * cpad]) : -1.0;
    }
    cluster.sync();  // A: slots published
    if (tid == 0) {
      double gb = -1.0;
      int gi = 0x7fffffff;
      for (int q = 0; q < cs; ++q) {
        const PanelSlot* s = cluster.map_shared_rank(&slot, q);
        const double v = s->val;
        const int r = s->row;
        if (v > gb || (v == gb && r < gi)) gb = v, gi = r;
      }
      const PanelSlot* sd = cluster.map_shared_rank(&slot, j / chunk);
      const double diag = sd->diag;
      int p = diag >= kPivThreshold * gb ? j : gi;
      if (!(gb >= kSingularTiny)) {
        if (rank == 0) atomicOr(&flags[0], 1);
        p = j;
      }
      if (rank == 0) {
        ipiv[F.start + k + j] = k + p;
        if (p != j) atomicAdd(&flags[1], 1);
      }
      piv_s = p;
    }
    __syncthreads();
    const int p = piv_s;
    const int op = p / chunk, oj = j / chunk;
    if (tid < w) {
      const double* rp = cluster.map_shared_rank(pan, op);
      urow[tid] = rp[(p - op * chunk) + tid * cpad];
      if (p != j && rank == op) {
        const double* rj = cluster.map_shared_rank(pan, oj);
        tmprow[tid] = rj[(j - oj * chunk) + tid * cpad];
      }
    }
    cluster.sync();  // B: everybody has read the rows it needs
    if (tid < w) {
      if (rank == oj) pan[(j - r0) + tid * cpad] = urow[tid];
      if (p != j && rank == op) pan[(p - r0) + tid * cpad] = tmprow[tid];
    }
    __syncthreads();
    const double ujj = urow[j];
    for (int i = max(0, j + 1 - r0) + tid; i < nloc; i += NT) {
      const double l = pan[i + j * cpad] / ujj;
      pan[i + j * cpad] = l;
      for (int c = j + 1; c < w; ++c) pan[i + c * cpad] -= l * urow[c];
    }
    __syncthreads();
  }
  for (int c = warp; c < w; c += NT / 32)
    for (int i = lane; i < nloc; i += 32) g[(k + r0 + i) + (int64_t)(k + c) * F.ld] = pan[i + c * cpad];
  cluster.sync();
  if (rank == 0) {
    // gather the w x w diagonal block, build inv(L11) (unit lower) and inv(U11)
    for (int idx = tid; idx < w * w; idx += NT) {
      const int r = idx % w, c = idx / w;
      const int o = r / chunk;
      const double* rp = cluster.map_shared_rank(pan, o);
      T[r + c * kNB] = rp[(r - o * chunk) + c * cpad];
    }
    __syncthreads();
    double* invL = scratch + (int64_t)F.scratch * 2 * kNB * kNB;
    double* invU = invL + kNB * kNB;
    if (tid < kNB) {
      const int c = tid;
      // column c of inv(L): X[c][c] = 1, X[i][c] = -sum_{t=c}^{i-1} L[i][t] X[t][c]
      double x[kNB];
      for (int i = 0; i < kNB; ++i) x[i] = 0.0;
      if (c < w) {
        x[c] = 1.0;
        for (int i = c + 1; i < w; ++i) {
          double s = 0.0;
          for (int t = c; t < i; ++t) s += T[i + t * kNB] * x[t];
          x[i] = -s;
        }
      }
      for (int i = 0; i < kNB; ++i) invL[i + c * kNB] = x[i];
      // column c of inv(U): X[c][c] = 1/U[c][c]; X[i][c] = -(sum_{t=i+1}^{c} U[i][t] X[t][c]) / U[i][i]
      for (int i = 0; i < kNB; ++i) x[i] = 0.0;
      if (c < w) {
        x[c] = 1.0 / T[c + c * kNB];
        for (int i = c - 1; i >= 0; --i) {
          double s = 0.0;
          for (int t = i + 1; t <= c; ++t) s += T[i + t * kNB] * x[t];
          x[i] = -s / T[i + i * kNB];
        }
      }
      for (int i = 0; i < kNB; ++i) invU[i + c * kNB] = x[i];
    }
  }
  cluster.sync();  // keep every CTA's shared memory alive until rank 0 is done
}

// ---------------------------------------------------------------------------
// Row swaps outside the panel, U12 = inv(L11) A12, L_cb = A_cb inv(U11).
// grid: (ncolblocks + nrowblocks, nfronts), block 256.
__global__ void __launch_bounds__(256) panel_apply(const FrontDev* __restrict__ fronts,
                                                  const int32_t* __restrict__ list, int k,
                                                  double* __restrict__ pool,
                                                  const int32_t* __restrict__ ipiv,
                                                  const double* __restrict__ scratch) {
  __shared__ double inv[kNB * kNB];
  const FrontDev F = fronts[list[blockIdx.y]];
  const int np = F.npiv, nf = F.nf;
  const int w = min(kNB, np - k);
  const int ncolb = (nf + 31) / 32;
  const int ncb = nf - np;
  const int nrowb = (ncb + 255) / 256;
  if ((int)blockIdx.x >= ncolb + nrowb) return;
  const double* invL = scratch + (int64_t)F.scratch * 2 * kNB * kNB;
  const double* invU = invL + kNB * kNB;
  double* g = pool + F.off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if ((int)blockIdx.x < ncolb) {
    for (int i = tid; i < kNB * kNB; i += 256) inv[i] = invL[i];
    __syncthreads();
    const int myp = lane < w ? ipiv[F.start + k + lane] : k + lane;
    const unsigned swaps = __ballot_sync(0xffffffffu, lane < w && myp != k + lane);
    for (int cc = warp; cc < 32; cc += 8) {
      const int c = blockIdx.x * 32 + cc;
      if (c >= nf || (c >= k && c < k + w)) continue;
      double* col = g + (int64_t)c * F.ld;
      if (swaps) {
        if (lane == 0)
          for (int jj = 0; jj < w; ++jj) {
            const int p = __ldg(&ipiv[F.start + k + jj]);
            if (p != k + jj) {
              const double t = col[k + jj];
              col[k + jj] = col[p];
              col[p] = t;
            }
          }
        __syncwarp();
      }
      if (c >= k + w) {
        const double a = lane < w ? col[k + lane] : 0.0;
        double s = 0.0;
        for (int t = 0; t < w; ++t) s += inv[lane + t * kNB] * __shfl_sync(0xffffffffu, a, t);
        if (lane < w) col[k + lane] = s;
      }
    }
  } else {
    for (int i = tid; i < kNB * kNB; i += 256) inv[i] = invU[i];
    __syncthreads();
    const int r = np + (blockIdx.x - ncolb) * 256 + tid;
    if (r >= nf) return;
    double a[kNB];
#pragma unroll
    for (int t = 0; t < kNB; ++t) a[t] = t < w ? g[r + (int64_t)(k + t) * F.ld] : 0.0;
#pragma unroll
    for (int i = 0; i < kNB; ++i) {
      if (i >= w) break;
      double s = 0.0;
#pragma unroll
      for (int t = 0; t <= i; ++t) s += a[t] * inv[t + i * kNB];
      g[r + (int64_t)(k + i) * F.ld] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// Trailing update A22 -= L21 U12 with DMMA (mma.sync.m16n8k4 f64).
// grid: (tiles, nfronts), block 128 (2x2 warps of 32x32), tile 64x64, K = w <= 32.
constexpr int kTS = 64;
constexpr int kSP = kTS + 4;  // padded smem stride (conflict-free fragment loads)

__device__ __forceinline__ void dmma16n8k4(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

__global__ void __launch_bounds__(128) schur_dmma(const FrontDev* __restrict__ fronts,
                                                 const int32_t* __restrict__ list, int k,
                                                 double* __restrict__ pool) {
  __shared__ double As[kNB * kSP];  // As[kk][m]
  __shared__ double Bs[kNB * kSP];  // Bs[kk][n]
  const FrontDev F = fronts[list[blockIdx.y]];
  const int np = F.npiv, nf = F.nf;
  const int w = min(kNB, np - k);
  const int c0 = k + w;
  const int Tn = nf - c0;
  if (Tn <= 0) return;
  const int nt = (Tn + kTS - 1) / kTS;
  if ((int)blockIdx.x >= nt * nt) return;
  const int tm = blockIdx.x % nt, tn = blockIdx.x / nt;
  const int m0 = c0 + tm * kTS, n0 = c0 + tn * kTS;
  double* g = pool + F.off;
  const int64_t ld = F.ld;
  const int tid = threadIdx.x;
  // A tile: L[m0 + m, k + kk]
  for (int idx = tid; idx < kNB * kTS; idx += 128) {
    const int kk = idx / kTS, m = idx % kTS;
    As[kk * kSP + m] = (kk < w && m0 + m < nf) ? g[(m0 + m) + (int64_t)(k + kk) * ld] : 0.0;
  }
  // B tile: U[k + kk, n0 + n]
  for (int idx = tid; idx < kNB * kTS; idx += 128) {
    const int kk = idx % kNB, n = idx / kNB;
    Bs[kk * kSP + n] = (kk < w && n0 + n < nf) ? g[(k + kk) + (int64_t)(n0 + n) * ld] : 0.0;
  }
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  const int gid = lane >> 2, tig = lane & 3;
  double acc[2][4][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][b][e] = 0.0;
  const int ksteps = (w + 3) / 4;
  for (int ks = 0; ks < ksteps; ++ks) {
    const int kr = ks * 4 + tig;
    double af[2][2], bf[4];
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      af[a][0] = As[kr * kSP + wm + a * 16 + gid];
      af[a][1] = As[kr * kSP + wm + a * 16 + gid + 8];
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) bf[b] = Bs[kr * kSP + wn + b * 8 + gid];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma16n8k4(acc[a][b], af[a][0], af[a][1], bf[b]);
  }
  // C fragment: c0,c1 -> (row gid, cols 2tig, 2tig+1); c2,c3 -> row gid+8
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = m0 + wm + a * 16 + gid + (e >> 1) * 8;
        const int c = n0 + wn + b * 8 + 2 * tig + (e & 1);
        if (r < nf && c < nf) g[r + c * ld] -= acc[a][b][e];
      }
}

// ---------------------------------------------------------------------------
// Host orchestration.
namespace {

int div_up(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace

namespace {

// Destination of every CSR entry in the front pool (the symbolic scatter map):
// entry (i, j) goes to the front owning pivot min(p(i), p(j)), at the local
// positions of p(i), p(j) in its sorted row list. One warp per matrix row.
__global__ void scatter_map_k(int64_t n, const int64_t* __restrict__ rowptr,
                              const int32_t* __restrict__ col, const int32_t* __restrict__ iperm,
                              const int32_t* __restrict__ owner, const FrontDev* __restrict__ fronts,
                              const int32_t* __restrict__ rows, int64_t* __restrict__ dst, int* bad) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw) {
    const int32_t ni = iperm[i];
    for (int64_t k = rowptr[i] + lane; k < rowptr[i + 1]; k += 32) {
      const int32_t nj = iperm[col[k]];
      const FrontDev F = fronts[owner[min(ni, nj)]];
      const int32_t* rb = rows + F.rows_off;
      int a = 0, b = F.nf;
      while (a < b) {
        const int m = (a + b) >> 1;
        if (rb[m] < ni) a = m + 1; else b = m;
      }
      const int pi = a;
      a = 0;
      b = F.nf;
      while (a < b) {
        const int m = (a + b) >> 1;
        if (rb[m] < nj) a = m + 1; else b = m;
      }
      const int pj = a;
      if (pi == F.nf || rb[pi] != ni || pj == F.nf || rb[pj] != nj) {
        atomicExch(bad, 1);
        dst[k] = 0;
      } else {
        dst[k] = F.off + pi + static_cast<int64_t>(pj) * F.ld;
      }
    }
  }
}

}  // namespace

FactorEngine::FactorEngine(const Symbolic& s, int64_t n_, const int64_t* rowptr,
                           const int32_t* col, const double* aval, const int64_t* rowptr_dev,
                           const int32_t* col_dev)
    : sym(s), n(n_) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    fail(errc::config, "no CUDA device: the B200 path has no CPU fallback");
  RQB_CUDA(cudaGetDevice(&device));
  cudaDeviceProp prop;
  RQB_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10) fail(errc::config, "an sm_100a (Blackwell) device is required");
  RQB_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  RQB_CUDA(cudaEventCreate(&ev0));
  RQB_CUDA(cudaEventCreate(&ev1));
  nnz = rowptr[n];
  SetupTrace tr("FactorEngine");
  if (n != sym.n) fail(errc::dimension, "matrix size differs from the symbolic analysis");

  // Front descriptors, extend-add inverse maps, launch plans.
  const int nfr = static_cast<int>(sym.fronts.size());
  fronts_h.resize(nfr);
  std::vector<int32_t> inv;
  for (int f = 0; f < nfr; ++f) {
    const Front& F = sym.fronts[f];
    FrontDev& D = fronts_h[f];
    D.off = F.off;
    D.rows_off = F.rows_off;
    D.cbvec_off = F.cbvec_off;
    D.nf = F.nf;
    D.npiv = F.npiv;
    D.ld = F.ld;
    D.start = F.start;
    D.nchild = static_cast<int32_t>(F.children.size());
    if (D.nchild > 2) fail(errc::generic, "front with more than two children");
    D.child0 = D.nchild > 0 ? F.children[0] : -1;
    D.child1 = D.nchild > 1 ? F.children[1] : -1;
    D.scratch = -1;
    D.rel_off = 0;
    D.inv_off = static_cast<int64_t>(inv.size());
    const int32_t* prow = sym.rows.data() + F.rows_off;
    for (int32_t c : F.children) {
      const Front& C = sym.fronts[c];
      const int32_t* crow = sym.rows.data() + C.rows_off;
      // child CB rows are a sorted subset of the parent's rows
      std::vector<int32_t> m(F.nf, -1);
      int pi = 0;
      fronts_h[c].rel_off = static_cast<int64_t>(rel_h.size());
      for (int t = C.npiv; t < C.nf; ++t) {
        while (pi < F.nf && prow[pi] < crow[t]) ++pi;
        if (pi == F.nf || prow[pi] != crow[t]) fail(errc::generic, "child CB row missing in parent");
        m[pi] = t;
        rel_h.push_back(pi);
      }
      inv.insert(inv.end(), m.begin(), m.end());
    }
  }
  plans.resize(sym.level_fronts.size());
  std::vector<int32_t> lists;
  auto push_list = [&](const std::vector<int32_t>& v) {
    const int64_t o = static_cast<int64_t>(lists.size());
    lists.insert(lists.end(), v.begin(), v.end());
    return o;
  };
  for (size_t l = 0; l < sym.level_fronts.size(); ++l) {
    LevelPlan& P = plans[l];
    int slot = 0;
    for (int32_t f : sym.level_fronts[l]) {
      const Front& F = sym.fronts[f];
      P.all.push_back(f);
      P.solve_maxnf = std::max(P.solve_maxnf, F.nf);
      if (!F.children.empty()) {
        P.with_kids.push_back(f);
        P.ea_maxnf = std::max(P.ea_maxnf, F.nf);
      }
      if (F.npiv == 0) continue;
      if (F.nf <= kSmallNf) {
        P.small.push_back(f);
        P.small_nf = std::max(P.small_nf, F.nf);
      } else {
        P.big.push_back(f);
        fronts_h[f].scratch = slot++;
        P.big_maxnf = std::max(P.big_maxnf, F.nf);
        P.big_maxrows = std::max(P.big_maxrows, F.npiv);
        P.big_maxpanels = std::max(P.big_maxpanels, div_up(F.npiv, kNB));
      }
    }
    nscratch = std::max<int64_t>(nscratch, slot);
    P.big_cluster = std::min(8, std::max(1, div_up(P.big_maxrows, kPanelRowsMax)));
    if (div_up(P.big_maxrows, P.big_cluster) > kPanelRowsMax)
      fail(errc::config, "front too large for the 8-CTA panel cluster");
    P.off_small = push_list(P.small);
    P.off_big = push_list(P.big);
    P.off_kids = push_list(P.with_kids);
    P.off_all = push_list(P.all);
    P.panel_fronts.resize(P.big_maxpanels);
    P.off_panel.resize(P.big_maxpanels);
    for (int s = 0; s < P.big_maxpanels; ++s) {
      for (int32_t f : P.big)
        if (s * kNB < sym.fronts[f].npiv) P.panel_fronts[s].push_back(f);
      P.off_panel[s] = push_list(P.panel_fronts[s]);
    }
  }
  tr.mark("fronts+plans");
  d_pool.alloc(sizeof(double) * sym.pool);
  if (aval)
    d_aval.upload(aval, sizeof(double) * nnz, stream);
  else
    d_aval.alloc(sizeof(double) * nnz);  // values arrive by set_values_device
  d_rows.upload(sym.rows.data(), sizeof(int32_t) * sym.rows.size(), stream);
  d_fronts.upload(fronts_h.data(), sizeof(FrontDev) * fronts_h.size(), stream);
  if (inv.empty()) inv.push_back(-1);
  if (lists.empty()) lists.push_back(0);
  d_inv.upload(inv.data(), sizeof(int32_t) * inv.size(), stream);
  if (rel_h.empty()) rel_h.push_back(0);
  d_rel.upload(rel_h.data(), sizeof(int32_t) * rel_h.size(), stream);
  d_lists.upload(lists.data(), sizeof(int32_t) * lists.size(), stream);
  d_ipiv.alloc(sizeof(int32_t) * n);
  d_scratch.alloc(sizeof(double) * std::max<int64_t>(1, nscratch) * 2 * kNB * kNB);
  d_flags.alloc(sizeof(int) * 4);
  d_arrived.alloc(sizeof(int));
  d_y.alloc(sizeof(double) * n);
  d_xnew.alloc(sizeof(double) * n);
  d_cbvec.alloc(sizeof(double) * std::max<int64_t>(1, sym.cbvec));
  d_perm.upload(sym.perm.data(), sizeof(int32_t) * n, stream);
  tr.mark("uploads");
  {
    // scatter map on the device (pattern from the caller's device copy when given)
    std::vector<int32_t> owner(n);
    for (size_t f = 0; f < sym.fronts.size(); ++f)
      for (int k = 0; k < sym.fronts[f].npiv; ++k) owner[sym.fronts[f].start + k] = static_cast<int32_t>(f);
    DeviceBuffer d_rp, d_cl, d_own, d_ip, d_bad;
    if (!rowptr_dev) {
      d_rp.upload(rowptr, sizeof(int64_t) * (n + 1), stream);
      rowptr_dev = d_rp.as<int64_t>();
    }
    if (!col_dev) {
      d_cl.upload(col, sizeof(int32_t) * std::max<int64_t>(nnz, 1), stream);
      col_dev = d_cl.as<int32_t>();
    }
    d_own.upload(owner.data(), sizeof(int32_t) * n, stream);
    d_ip.upload(sym.iperm.data(), sizeof(int32_t) * n, stream);
    d_bad.alloc(sizeof(int));
    RQB_CUDA(cudaMemsetAsync(d_bad.p, 0, sizeof(int), stream));
    d_qdst.alloc(sizeof(int64_t) * std::max<int64_t>(nnz, 1));
    const int64_t blocks = std::min<int64_t>(div_up(n, 8), 148 * 16);
    if (n > 0)
      scatter_map_k<<<static_cast<unsigned>(std::max<int64_t>(blocks, 1)), 256, 0, stream>>>(
          n, rowptr_dev, col_dev, d_ip.as<int32_t>(), d_own.as<int32_t>(), d_fronts.as<FrontDev>(),
          d_rows.as<int32_t>(), d_qdst.as<int64_t>(), d_bad.as<int>());
    RQB_CUDA(cudaGetLastError());
    int bad = 0;
    RQB_CUDA(cudaMemcpyAsync(&bad, d_bad.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
    RQB_CUDA(cudaStreamSynchronize(stream));
    if (bad) fail(errc::dimension, "matrix entry outside the symbolic front structure");
  }
  tr.mark("scatter_map");
  rqb_solve_prepare(*this);
  tr.mark("solve_prepare");
  {
    const char* mode = std::getenv("RQB_FACTOR");
    use_dag = !(mode && std::string(mode) == "level");
  }
  if (use_dag) rqb_dag_build(*this);
  tr.mark("dag_build");
  RQB_CUDA(cudaFuncSetAttribute(front_lu_smem<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmallNf * kSmallNf * 8));
  RQB_CUDA(cudaFuncSetAttribute(panel_lu<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (kPanelRowsMax + 1) * kNB * 8));
  RQB_CUDA(cudaFuncSetAttribute(panel_lu<256>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  RQB_CUDA(cudaStreamSynchronize(stream));
}

FactorEngine::~FactorEngine() {
  if (graph_factor_exec) cudaGraphExecDestroy(graph_factor_exec);
  if (graph_factor) cudaGraphDestroy(graph_factor);
  if (stream_up) cudaStreamDestroy(stream_up);
  if (ev_up) cudaEventDestroy(ev_up);
  if (h_marks) cudaFreeHost(h_marks);
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  if (stream) cudaStreamDestroy(stream);
}

void FactorEngine::set_values(const double* aval) {
  RQB_CUDA(cudaMemcpyAsync(d_aval.p, aval, sizeof(double) * nnz, cudaMemcpyHostToDevice, stream));
}

void FactorEngine::set_values_device(const double* aval_dev) {
  RQB_CUDA(cudaMemcpyAsync(d_aval.p, aval_dev, sizeof(double) * nnz, cudaMemcpyDeviceToDevice,
                           stream));
}

void FactorEngine::enqueue_factor(KernelTimer* kt) {
  int64_t launches = 0;
  auto B = [&](int kind) {
    if (kt) kt->begin(stream, kind);
  };
  auto E = [&]() {
    if (kt) kt->end(stream);
  };
  const FrontDev* fr = d_fronts.as<FrontDev>();
  const int32_t* lists = d_lists.as<int32_t>();
  double* pool = d_pool.as<double>();
  int32_t* ipiv = d_ipiv.as<int32_t>();
  int* flags = d_flags.as<int>();
  RQB_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * 4, stream));
  if (!(use_dag && dag_lazy)) {
    RQB_CUDA(cudaMemsetAsync(pool, 0, sizeof(double) * sym.pool, stream));
    B(0);
    scatter_original<<<std::min<int64_t>(div_up(nnz, 256), 148 * 16), 256, 0, stream>>>(
        d_aval.as<double>(), d_qdst.as<int64_t>(), nnz, pool);
    E();
    launches += 1;
  }
  if (use_dag) {
    B(6);
    rqb_dag_enqueue(*this);
    E();
    B(4);
    rqb_rowperm_enqueue(*this);
    E();
    launches += 3;
    RQB_CUDA(cudaGetLastError());
    launches_factor = launches;
    return;
  }
  for (const LevelPlan& P : plans) {
    if (!P.with_kids.empty()) {
      dim3 grid(div_up(P.ea_maxnf, 8), static_cast<unsigned>(P.with_kids.size()));
      B(1);
      extend_add<<<grid, dim3(32, 8), 0, stream>>>(fr, lists + P.off_kids, d_inv.as<int32_t>(), pool);
      E();
      ++launches;
    }
    if (!P.small.empty()) {
      const size_t smem = sizeof(double) * P.small_nf * P.small_nf;
      B(2);
      front_lu_smem<256><<<static_cast<unsigned>(P.small.size()), 256, smem, stream>>>(
          fr, lists + P.off_small, pool, ipiv, flags);
      E();
      ++launches;
    }
    for (int s = 0; s < P.big_maxpanels; ++s) {
      const int nfa = static_cast<int>(P.panel_fronts[s].size());
      const int32_t* lst = lists + P.off_panel[s];
      const int k = s * kNB;
      int maxr = 0, maxnf = 0, maxcb = 0;
      for (int32_t f : P.panel_fronts[s]) {
        maxr = std::max(maxr, sym.fronts[f].npiv - k);
        maxnf = std::max(maxnf, sym.fronts[f].nf);
        maxcb = std::max(maxcb, sym.fronts[f].nf - sym.fronts[f].npiv);
      }
      const int cs = std::min(8, std::max(1, div_up(maxr, kPanelRowsMax)));
      const int chunk = div_up(maxr, cs);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(nfa * cs);
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = sizeof(double) * (chunk | 1) * kNB;
      cfg.stream = stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      B(3);
      RQB_CUDA(cudaLaunchKernelEx(&cfg, panel_lu<256>, fr, lst, k, pool, ipiv, d_scratch.as<double>(),
                                  flags));
      E();
      dim3 ga(div_up(maxnf, 32) + div_up(maxcb, 256), nfa);
      B(4);
      panel_apply<<<ga, 256, 0, stream>>>(fr, lst, k, pool, ipiv, d_scratch.as<double>());
      E();
      const int tmax = maxnf - k - 1;
      launches += 2;
      if (tmax > 0) {
        const int nt = div_up(tmax, kTS);
        dim3 gs(nt * nt, nfa);
        B(5);
        schur_dmma<<<gs, 128, 0, stream>>>(fr, lst, k, pool);
        E();
        ++launches;
      }
    }
  }
  B(4);
  rqb_rowperm_enqueue(*this);
  E();
  launches += 2;
  RQB_CUDA(cudaGetLastError());
  launches_factor = launches;
}

void FactorEngine::factor_streamed(const double* aval) {
  static const bool off = std::getenv("RQB_STREAM_UPLOAD") && std::atoi(std::getenv("RQB_STREAM_UPLOAD")) == 0;
  if (!(use_dag && dag_lazy) || off || nnz < (1 << 20)) {
    set_values(aval);
    factor();
    return;
  }
  const int64_t kChunk = stream_chunk;
  const int nch = static_cast<int>(chunk_order.size());
  if (nch == 0) {
    set_values(aval);
    factor();
    return;
  }
  if (!stream_up) {
    RQB_CUDA(cudaStreamCreateWithFlags(&stream_up, cudaStreamNonBlocking));
    RQB_CUDA(cudaEventCreateWithFlags(&ev_up, cudaEventDisableTiming));
  }
  if (n_marks != nch) {
    if (h_marks) cudaFreeHost(h_marks);
    RQB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_marks), sizeof(int) * nch));
    for (int c = 0; c < nch; ++c) h_marks[c] = c + 1;
    n_marks = nch;
  }
  if (!graph_factor_exec) {  // first use: capture with the values resident
    set_values(aval);
    factor();
    return;
  }
  streaming = true;
  try {
    // everything enqueued so far (earlier solves read the factors, an earlier
    // factorization reads d_aval) precedes the first chunk
    RQB_CUDA(cudaMemsetAsync(d_arrived.p, 0, sizeof(int), stream));
    RQB_CUDA(cudaEventRecord(ev0, stream));  // last_ms: upload + factorization
    RQB_CUDA(cudaEventRecord(ev_up, stream));
    RQB_CUDA(cudaStreamWaitEvent(stream_up, ev_up, 0));
    // the graph first: its state-reset copies must not queue behind the chunks on a copy engine
    launch_factor_graph();
    for (int c = 0; c < nch; ++c) {
      const int64_t o = chunk_order[c] * kChunk, len = std::min<int64_t>(nnz, o + kChunk) - o;
      RQB_CUDA(cudaMemcpyAsync(d_aval.as<double>() + o, aval + o, sizeof(double) * len, cudaMemcpyHostToDevice,
                               stream_up));
      RQB_CUDA(cudaMemcpyAsync(d_arrived.p, h_marks + c, sizeof(int), cudaMemcpyHostToDevice, stream_up));
    }
    static const bool dbg = std::getenv("RQB_STREAM_DEBUG") != nullptr;
    if (dbg) {
      cudaEvent_t e;
      RQB_CUDA(cudaEventCreate(&e));
      RQB_CUDA(cudaEventRecord(e, stream_up));
      RQB_CUDA(cudaEventSynchronize(e));
      float ms = 0;
      RQB_CUDA(cudaEventElapsedTime(&ms, ev0, e));
      std::fprintf(stderr, "[stream] upload of %d chunks done %.3f ms after the reset\n", nch, ms);
      cudaEventDestroy(e);
    }
    RQB_CUDA(cudaStreamSynchronize(stream_up));
  } catch (...) {
    streaming = false;
    cudaStreamSynchronize(stream_up);
    cudaStreamSynchronize(stream);
    throw;
  }
  streaming = false;
  finish_factor();
}

void FactorEngine::factor() {
  RQB_CUDA(cudaMemsetAsync(d_arrived.p, 0x7f, sizeof(int), stream));  // values resident
  launch_factor_graph();
  finish_factor();
}

void FactorEngine::launch_factor_graph() {
  if (!graph_factor_exec) {
    RQB_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    enqueue_factor();
    RQB_CUDA(cudaStreamEndCapture(stream, &graph_factor));
    RQB_CUDA(cudaGraphInstantiate(&graph_factor_exec, graph_factor, 0));
  }
  if (!streaming) RQB_CUDA(cudaEventRecord(ev0, stream));
  RQB_CUDA(cudaGraphLaunch(graph_factor_exec, stream));
  RQB_CUDA(cudaEventRecord(ev1, stream));
}

void FactorEngine::finish_factor() {
  int flags[4];
  RQB_CUDA(cudaMemcpyAsync(flags, d_flags.p, sizeof(flags), cudaMemcpyDeviceToHost, stream));
  RQB_CUDA(cudaStreamSynchronize(stream));
  float ms = 0;
  RQB_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
  last_ms = ms;
  last_swaps = flags[1];
  if (flags[2])
    fail(errc::solver, std::string("factorization task DAG stalled (watchdog): ") + rqb_dag_stall_report(*this));
  if (flags[0]) fail(errc::singular, "Q(sigma) is numerically singular: every pivot candidate below 1e-300");
}

}  // namespace rqb

namespace rqb {

void KernelTimer::begin(cudaStream_t s, int kind) {
  cudaEvent_t a, b;
  RQB_CUDA(cudaEventCreate(&a));
  RQB_CUDA(cudaEventCreate(&b));
  RQB_CUDA(cudaEventRecord(a, s));
  ev.push_back({a, b});
  kinds.push_back(kind);
}

void KernelTimer::end(cudaStream_t s) { RQB_CUDA(cudaEventRecord(ev.back().second, s)); }

void KernelTimer::collect(double* ms, int64_t* count, int nkinds) {
  for (size_t i = 0; i < ev.size(); ++i) {
    float t = 0;
    RQB_CUDA(cudaEventSynchronize(ev[i].second));
    RQB_CUDA(cudaEventElapsedTime(&t, ev[i].first, ev[i].second));
    if (kinds[i] < nkinds) ms[kinds[i]] += t, count[kinds[i]] += 1;
    cudaEventDestroy(ev[i].first);
    cudaEventDestroy(ev[i].second);
  }
  ev.clear();
  kinds.clear();
}

void FactorEngine::profile(double* ms, int64_t* count, double* flops) {
  for (int k = 0; k < kFactorKinds; ++k) ms[k] = 0, count[k] = 0, flops[k] = 0;
  KernelTimer kt;
  enqueue_factor(&kt);
  kt.collect(ms, count, kFactorKinds);
  // algorithmic work per kernel class (real flops; scatter/extend-add: bytes)
  double bytes_scatter = 16.0 * nnz + 8.0 * nnz;  // read value + index, write entry
  double ea = 0;
  for (const Front& F : sym.fronts)
    if (F.parent >= 0) {
      const double ncb = F.nf - F.npiv;
      ea += 16.0 * ncb * ncb;  // read the child's block, read+write the parent entry (~)
    }
  flops[0] = bytes_scatter;
  flops[1] = ea;
  for (const Front& F : sym.fronts) {
    double flu = 0;
    for (int k = 0; k < F.npiv; ++k) {
      const double r = F.nf - k - 1.0;
      flu += r + 2.0 * r * r;
    }
    if (F.npiv == 0) continue;
    if (F.nf <= kSmallNf) {
      flops[2] += flu;
      continue;
    }
    double sch = 0;
    for (int k = 0; k < F.npiv; k += kNB) {
      const double w = std::min(kNB, F.npiv - k);
      const double t = F.nf - k - w;
      sch += 2.0 * w * t * t;
    }
    flops[5] += sch;
    flops[3] += flu - sch;  // panel LU + TRSM (panel_apply shares this count)
  }
  if (use_dag) {
    flops[6] = sym.flops_lu;  // the persistent kernel does the whole factorization
    flops[2] = flops[3] = flops[5] = 0;
  }
}

}  // namespace rqb
