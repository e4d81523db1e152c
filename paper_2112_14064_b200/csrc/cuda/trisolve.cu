// SPDX-License-Identifier: Apache-2.0
// Multifrontal forward/backward substitution (solve_factored)
// as two persistent dataflow kernels (one launch per sweep) over the
// device-resident fronts.
//
// Work items are 64-row blocks of a front. Readiness is tracked per front:
// when a front becomes ready (forward: its children completed; backward: the
// nearest ancestor with pivots completed) one thread pushes ALL its items, in
// order, on a FIFO ready queue; persistent CTAs claim queue slots in order.
// Inside a front the items are left-looking and wait only for earlier items
// of the same front (earlier queue slots, hence already claimed and running),
// consuming each finished block as soon as it is published: the chain per
// block is one 64x64 GEMV + one triangle, the L/U loads of the next block are
// prefetched while waiting. No level barriers, one launch per sweep.
//   forward   w = b(pivot rows, after the front's net row permutation) +
//             children's contribution vectors (gather, atomic-free);
//             s = L[rows, 0:j) y; pivot block: unit-lower 64x64 triangle in
//             shared memory -> y; contribution rows: w - s -> the front's
//             contribution vector for the parent.
//   backward  s = y - U[rows, cb] x_cb (ancestors' solution) - U[rows, later] x;
//             upper 64x64 triangle; writes x (ND order for descendants, caller
//             order scaled, and the fused r_l = s r_u + v_u of apply_operator).
// Loads of data produced inside the sweep use ld.global.cg (L1 bypass);
// publication is __threadfence + atomic.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "device.cuh"

namespace rqb {

constexpr int kRB = 64;   // rows per item
constexpr int kST = 256;  // threads per CTA

// One work item: up to 64 rows of a front, with the front fields it needs
// (one 64-byte record; the item's first instruction loads need no further
// indirection).
struct SolveItem {
  int64_t goff;                   // front's pool offset (doubles)
  int32_t front, r0, nr, blk;     // local rows [r0, r0+nr); pivot-block index, -1 contribution rows
  int32_t ld, np, nf, start;
  int32_t npb, ncbb, parent, rows_off;
  int32_t cbvec_off, ech_off, nech, doff;  // doff: the front's first diagonal-inverse block
};

struct SweepArgs {
  const SolveItem* items;
  int nitems;
  int* deps;      // per front: unfinished predecessor fronts
  int* queue;
  int* qctl;      // {head, tail}
  int* done;      // items finished (termination of pop_item)
  int* pub;       // per front: pivot blocks published (forward: first first; backward: last first)
  int* fin;       // per front: forward items finished
  int fwd;        // 1 forward, 0 backward (item layout of front_ready)
  int win;        // window of pivot blocks in the queue per front (kWin; RQB_WIN_F / RQB_WIN_B)
  const int32_t* fbase;  // per front: first item of this sweep
  const int32_t* fcnt;   // per front: items of this sweep
  const int32_t* npb;    // per front: pivot blocks (forward window: 0 for whole fronts)
  const int32_t* npart;  // backward: per front, contribution-column partial items ahead of its blocks
  int* pdone;            // backward: per front, partial items finished
  double* bpart;         // backward: partial sums U[blk rows, chunk] x_chunk (64 per partial item)
  const int32_t* ech;
  const int4* gsrc;      // forward gather sources per front row {b, child0 cb, child1 cb, -}
  const double* pool;
  const double* dinv;    // diagonal-block inverses (FactorEngine::d_dinv)
  const int32_t* perm;
  const int32_t* rows;
  const double* b;
  double* y;
  double* cbvec;
  double* xnew;
  double* xout;
  double scale;
  const double* vu;
  double sigma;
  double* xl_out;
  unsigned long long* trace;  // development trace (RQB_SOLVE_TRACE): per item 4 timestamps, SM, ns waited
  int* stall;                 // watchdog flag (persistent, checked by the host at its sync points)
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define RQB_TRACE(k)                                                       \
  if (A.trace && tid == 0) {                                               \
    A.trace[8 * (size_t)it + (k)] = gtime();                               \
  }

// Solution entries of pivot blocks are published by value: the solve resets
// y and x to an all-ones bit pattern (a NaN no FP64 operation produces; NaN
// results are canonical) and a waiting item polls the entries of the block it
// needs directly (relaxed loads of relaxed stores, 8-byte single-copy atomic):
// no fence or flag round trip on the chain of pivot blocks. The per-front
// counters stay for everything off the chain (windows, earlier blocks).
constexpr long long kUnset = -1LL;
__device__ __forceinline__ void st_relaxed(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Items enter the queue through a window of kWin pivot blocks: item v of a
// front (forward: pivot block v, v == npb stands for all contribution items;
// backward: the v-th block from the end) is pushed when the front becomes
// ready (v < kWin) or when the front's item v - kWin publishes. An item then
// waits for at most kWin - 1 blocks instead of holding a CTA through the
// whole pivot chain, yet starts early enough to stream the blocks published
// before it (measured: 32; 8 leaves the chain of the large top fronts waiting
// on the streaming). Pushes of one front happen in item order, so every wait
// targets an earlier queue slot (deadlock freedom of the FIFO claim order).
constexpr int kWin = 32;
constexpr int kStage = 1024;  // staged solution entries per round (8 KB)
// Fronts with at most kWholeNpb pivot blocks and kWholeCb contribution rows
// are one item per sweep (a single CTA walks the whole front, its y / x kept
// in shared memory): no inter-CTA publication latency on the many small
// fronts near the leaves.
constexpr int kWholeNpb = 2;
constexpr int kWholeCb = kStage - kWholeNpb * kRB;
constexpr int kWhole = -2;  // SolveItem::blk of a whole-front item
// Backward items of fronts with more than kCbChunk contribution columns are
// split: per pivot block, one partial item per kCbChunk columns (U[blk rows,
// chunk] x_chunk into bpart, no waits) ahead of the block item, which then only
// streams the later pivot blocks and adds its partials before the triangle.
constexpr int kCbChunk = 256;
constexpr int kPart = -3;  // SolveItem::blk of a partial item (cbvec_off/ncbb: column range, ech_off: slot)

__device__ __forceinline__ void push_items(const SweepArgs& A, int i0, int n) {
  if (n <= 0) return;
  const int slot = atomicAdd(&A.qctl[1], n);
  for (int i = 0; i < n; ++i) atomicExch(&A.queue[slot + i], i0 + i);
}

// push virtual items [v0, v1] of front f (clipped to what exists); with keep,
// the first of them is handed to the calling CTA instead (it never waits:
// nothing of its front precedes it), the rest go on the queue
__device__ __forceinline__ void push_window(const SweepArgs& A, int f, int v0, int v1, int* keep = nullptr) {
  const int npb = A.npb[f], base = A.fbase[f];
  int i0, n;
  if (A.fwd) {
    v1 = min(v1, npb);
    if (v0 > v1) return;
    const int end = v1 == npb ? base + A.fcnt[f] : base + v1 + 1;
    i0 = base + v0;
    n = end - i0;
  } else {  // [partial items] then the pivot blocks, last first; the partials enter with the window
    const int npart = A.npart[f];
    v1 = min(v1, npb - 1);
    if (v0 > v1) return;
    i0 = base + npart + v0;
    n = v1 - v0 + 1;
    if (v0 == 0) {
      i0 = base;
      n += npart;
    }
  }
  if (n <= 0) return;
  if (keep) {
    *keep = i0;
    ++i0;
    --n;
  }
  push_items(A, i0, n);
}

// one predecessor front of f finished; the last one opens f's window
__device__ __forceinline__ void front_ready(const SweepArgs& A, int f, int* keep = nullptr) {
  if (atomicSub(&A.deps[f], 1) == 1) {
    __threadfence();
    push_window(A, f, 0, A.win - 1, keep);
  }
}

// forward: one item of a child of f finished (deps counts the children's items);
// the acq_rel atomic publishes this CTA's contribution vector (ordered by the
// preceding barrier) and acquires the other items' on the last arrival
__device__ __forceinline__ void item_done_fwd(const SweepArgs& A, int f, int* keep) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], -1;" : "=r"(old) : "l"(A.deps + f) : "memory");
  if (old == 1) {
    __threadfence();
    push_window(A, f, 0, A.win - 1, keep);
  }
}

// Spin waits give up after kSweepStallNs (a dependency that never resolves is
// a bug): the flag is raised, every CTA drains, the host reports the stall.
constexpr unsigned long long kSweepStallNs = 4000000000ull;
__device__ __forceinline__ bool stalled(const SweepArgs& A, unsigned long long& t0) {
  if (*((volatile int*)A.stall)) return true;
  const unsigned long long t = gtime();
  if (t0 == 0) t0 = t;
  if (t - t0 > kSweepStallNs) {
    atomicExch(A.stall, 1);
    return true;
  }
  return false;
}


// Warp 0: wait until entries [0, n) of v (n <= 64) are published, stage them
// in dst. Returns false if the watchdog fired.
__device__ __forceinline__ bool poll_block(const SweepArgs& A, const double* v, int n, double* dst, int lane) {
  unsigned long long t0 = 0;
  for (;;) {
    const double a = lane < n ? ld_relaxed(v + lane) : 0.0;
    const double b = lane + 32 < n ? ld_relaxed(v + lane + 32) : 0.0;
    const bool ok = __double_as_longlong(a) != kUnset && __double_as_longlong(b) != kUnset;
    if (__all_sync(0xffffffffu, ok)) {
      if (lane < n) dst[lane] = a;
      if (lane + 32 < n) dst[lane + 32] = b;
      return true;
    }
    int st = 0;
    if (lane == 0) {
      __nanosleep(20);
      st = stalled(A, t0);
    }
    if (__shfl_sync(0xffffffffu, st, 0)) return false;
  }
}

// Claim the next queue slot and wait for it; -1 once every item has finished
// (items kept by a CTA never pass through the queue, so the last claimed
// slots stay empty).
__device__ __forceinline__ int pop_item(const SweepArgs& A) {
  const int h = atomicAdd(&A.qctl[0], 1);
  if (h >= A.nitems) return -1;
  int t;
  unsigned long long t0 = 0;
  while ((t = ld_acquire(&A.queue[h])) < 0) {
    if (ld_acquire(A.done) >= A.nitems) return -1;
    __nanosleep(20);
    if (stalled(A, t0)) return -1;
  }
  return t;
}

// s += sum_{c in [cb, ce)} L[row, c] xs[c] for this thread's column class
// (c = grp mod 4): eight independent column loads in flight per iteration,
// each a 512-byte coalesced segment across the 64 rows of the item; the last
// (partial) iteration is predicated, not a serial tail of dependent loads.
__device__ __forceinline__ double stream_cols(const double* lp, int64_t ld, const double* xs, int cb, int ce,
                                              int grp) {
  double s0 = 0.0, s1 = 0.0;
  int c = cb + grp;
  for (; c + 28 < ce; c += 32) {
    double a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = lp[(int64_t)(c + 4 * u) * ld];
#pragma unroll
    for (int u = 0; u < 8; u += 2) {
      s0 += a[u] * xs[c + 4 * u];
      s1 += a[u + 1] * xs[c + 4 * u + 4];
    }
  }
  if (c < ce) {  // fewer than 8 columns of this class left: one predicated batch
    double a[7];
#pragma unroll
    for (int u = 0; u < 7; ++u) a[u] = c + 4 * u < ce ? lp[(int64_t)(c + 4 * u) * ld] : 0.0;
#pragma unroll
    for (int u = 0; u < 7; ++u)
      if (c + 4 * u < ce) s0 += a[u] * xs[c + 4 * u];
  }
  return s0 + s1;
}

// registers of one 64-column block (issued before the wait for it)
__device__ __forceinline__ void load_block(double (&r)[kRB / 4], const double* lp, int64_t ld, bool rowok, int c0,
                                           int c1, int grp) {
#pragma unroll
  for (int u = 0; u < kRB / 4; ++u) {
    const int c = c0 + grp + 4 * u;
    r[u] = (rowok && c < c1) ? lp[(int64_t)c * ld] : 0.0;
  }
}

// sum of r[u] xs[grp + 4u] over the cw valid columns of a block
__device__ __forceinline__ double fma_block(const double (&r)[kRB / 4], const double* xs, int cw, int grp) {
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < kRB / 4; ++u)
    if (grp + 4 * u < cw) s += r[u] * xs[grp + 4 * u];
  return s;
}

// Inverse of an item's diagonal tile into shared memory, padded to 64 x 64
// with zeros (rows/columns >= nr): forward inv(L11) with its unit diagonal,
// backward inv(U11). The tiles are contiguous nr x nr squares (diag_inverse),
// so this is one coalesced read; the substitution becomes a 64 x 64 product
// with no serial chain.
template <bool kUpper>
__device__ __forceinline__ void load_dinv(double* D, const double* src, int nr, int tid) {
  constexpr int kPer = kRB * kRB / kST;
  double v[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {  // every load in flight before the first store
    const int idx = tid + u * kST, r = idx & (kRB - 1), c = idx >> 6;
    v[u] = 0.0;
    if (r < nr && c < nr) {
      if (kUpper)
        v[u] = r <= c ? src[r + c * nr] : 0.0;
      else
        v[u] = r > c ? src[r + c * nr] : (r == c ? 1.0 : 0.0);
    }
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int idx = tid + u * kST;
    D[(idx & (kRB - 1)) + (idx >> 6) * (kRB + 1)] = v[u];
  }
}

// partial of one pivot block, summed in a fixed order (u ascending): the
// sweeps add these per-block partials in block order, so results do not
// depend on how publication rounds happened to group the blocks
__device__ __forceinline__ double block_dot(const double* lp, int64_t ld, const double* xs, int c0, int c1,
                                            int grp) {
  double r[kRB / 4];
  load_block(r, lp, ld, true, c0, c1, grp);
  return fma_block(r, xs + c0, c1 - c0, grp);
}

// diagonal tile solve in warp 0 (lane holds rows lane, lane + 32): v <- D v
// with D the tile's inverse; 64 broadcasts, two independent FMA chains per row
// (only the tile's nr columns: the padding of D is zero; small fronts near
// the leaves have 20-40 pivots)
__device__ __forceinline__ void tile_apply(const double* D, int lane, double& v0, double& v1, int nr = kRB) {
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll 8
  for (int c = 0; c < nr; c += 2) {
    const double x0 = __shfl_sync(0xffffffffu, c < 32 ? v0 : v1, c & 31);
    const double x1 = __shfl_sync(0xffffffffu, c < 32 ? v0 : v1, (c + 1) & 31);
    a0 += D[lane + c * (kRB + 1)] * x0;
    b0 += D[lane + 32 + c * (kRB + 1)] * x0;
    a1 += D[lane + (c + 1) * (kRB + 1)] * x1;
    b1 += D[lane + 32 + (c + 1) * (kRB + 1)] * x1;
  }
  v0 = a0 + a1;
  v1 = b0 + b1;
}

// L2 prefetch of a contiguous byte range (TMA bulk prefetch, 16-byte granules)
__device__ __forceinline__ void prefetch_l2(const void* p, size_t bytes) {
  uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  while (a < e) {
    const unsigned n = static_cast<unsigned>(e - a < (uintptr_t(1) << 20) ? e - a : (uintptr_t(1) << 20));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
    a += n;
  }
}

__device__ __forceinline__ void red_release(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// s_a, s_b += L[ra, c] y_c, L[rb, c] y_c over the columns c = grp mod 4 of
// [0, ne) (contribution rows of a whole-front item; two rows per thread, 8
// loads in flight per batch, the partial batch predicated)
__device__ __forceinline__ void stream_rows2(const double* g, int64_t ld, const double* ys, int ne, int ra, bool oka,
                                             int rb, bool okb, int grp, double& sa, double& sb) {
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
  for (int c = grp; c < ne; c += 16) {
    double la[4], lb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool okc = c + 4 * u < ne;
      la[u] = oka && okc ? g[ra + (int64_t)(c + 4 * u) * ld] : 0.0;
      lb[u] = okb && okc ? g[rb + (int64_t)(c + 4 * u) * ld] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; u += 2) {
      const double y0 = c + 4 * u < ne ? ys[c + 4 * u] : 0.0;
      const double y1 = c + 4 * u + 4 < ne ? ys[c + 4 * u + 4] : 0.0;
      a0 += la[u] * y0;
      a1 += la[u + 1] * y1;
      b0 += lb[u] * y0;
      b1 += lb[u + 1] * y1;
    }
  }
  sa = a0 + a1;
  sb = b0 + b1;
}

// Forward sweep over one whole front (at most kWholeNpb pivot blocks) by one
// CTA: w of every row gathered at once (b + the children's contribution
// vectors) into wy, pivot blocks y = inv(L11) (w - L10 y) in warp 0 (y
// replaces w in wy), then every
// contribution row w - L y with four lanes per row (column classes reduced by
// shuffles), 128 rows per pass, no barriers between passes.
__device__ __forceinline__ void fwd_whole(const SweepArgs& A, const SolveItem& I, const double* g, int64_t ld,
                                          double* D, double* wy, double (*part)[kRB], int tid) {
  const int np = I.np, nf = I.nf;
  if (tid == 0) {
    prefetch_l2(g, sizeof(double) * (size_t)np * ld);  // L columns: one contiguous range
    for (int blk = 1; blk < I.npb; ++blk) {            // the later tile inverses
      const int nr = min(np, blk * kRB + kRB) - blk * kRB;
      prefetch_l2(A.dinv + I.doff + (int64_t)kRB * kRB * blk, sizeof(double) * nr * nr);
    }
  }
  {
    constexpr int kQ = kStage / kST;
    int4 src[kQ];
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const int r = tid + q * kST;
      src[q] = r < nf ? __ldg(&A.gsrc[I.rows_off + r]) : make_int4(-1, -1, -1, 0);
    }
    // the first tile inverse travels with the gather table (one round trip
    // instead of two before the first triangle)
    if (I.npb > 0) load_dinv<false>(D, A.dinv + I.doff, min(np, kRB), tid);
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      double v = 0.0;
      if (src[q].x >= 0) v = A.b[src[q].x];
      if (src[q].y >= 0) v += __ldcg(&A.cbvec[src[q].y]);
      if (src[q].z >= 0) v += __ldcg(&A.cbvec[src[q].z]);
      if (tid + q * kST < nf) wy[tid + q * kST] = v;
    }
  }
  const int row = tid & (kRB - 1), grp = tid >> 6;
  if (I.npb == 0) __syncthreads();
  for (int blk = 0; blk < I.npb; ++blk) {
    const int r0 = blk * kRB, nr = min(np, r0 + kRB) - r0;
    if (blk > 0) load_dinv<false>(D, A.dinv + I.doff + (int64_t)kRB * kRB * blk, nr, tid);
    double s = 0.0;
    if (row < nr && r0 > 0) s = stream_cols(g + r0 + row, ld, wy, 0, r0, grp);
    part[grp][row] = s;
    __syncthreads();
    if (tid < 32) {
      double v0 = tid < nr ? wy[r0 + tid] - (part[0][tid] + part[1][tid] + part[2][tid] + part[3][tid]) : 0.0;
      double v1 = tid + 32 < nr ? wy[r0 + tid + 32] -
                                      (part[0][tid + 32] + part[1][tid + 32] + part[2][tid + 32] + part[3][tid + 32])
                                : 0.0;
      tile_apply(D, tid, v0, v1, nr);
      if (tid < nr) A.y[I.start + r0 + tid] = wy[r0 + tid] = v0;
      if (tid + 32 < nr) A.y[I.start + r0 + tid + 32] = wy[r0 + tid + 32] = v1;
    }
    __syncthreads();
  }
  const int rr = tid >> 2, cg = tid & 3;
  for (int p0 = np; p0 < nf; p0 += 2 * kRB) {
    const int ra = p0 + rr, rb = ra + kRB;
    double sa = 0.0, sb = 0.0;
    if (np > 0) stream_rows2(g, ld, wy, np, ra, ra < nf, rb, rb < nf, cg, sa, sb);
    sa += __shfl_xor_sync(0xffffffffu, sa, 1);
    sb += __shfl_xor_sync(0xffffffffu, sb, 1);
    sa += __shfl_xor_sync(0xffffffffu, sa, 2);
    sb += __shfl_xor_sync(0xffffffffu, sb, 2);
    if (cg == 0) {
      if (ra < nf) A.cbvec[I.cbvec_off + ra - np] = wy[ra] - sa;
      if (rb < nf) A.cbvec[I.cbvec_off + rb - np] = wy[rb] - sb;
    }
  }
  __syncthreads();  // every row written before thread 0 publishes
}

template <int kMinBlocks>
__global__ void __launch_bounds__(kST, kMinBlocks) fwd_sweep(SweepArgs A) {
  __shared__ double D[kRB * (kRB + 1)];
  __shared__ double stg[kStage];  // staged y (whole-front items: the front's own y)
  __shared__ double part[4][kRB];
  __shared__ double wv[kRB];
  __shared__ int item_s, avail_s, keep_s, staged_s;
  const int tid = threadIdx.x, row = tid & (kRB - 1), grp = tid >> 6;
  if (tid == 0) keep_s = -1;
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      const unsigned long long tp = A.trace ? gtime() : 0;
      item_s = keep_s >= 0 ? keep_s : pop_item(A);
      keep_s = -1;
      if (A.trace && item_s >= 0) A.trace[8 * (size_t)item_s + 4] = tp;  // pop began (whole items: slot 4 free)
    }
    __syncthreads();
    const int it = item_s;
    if (it < 0) return;
    RQB_TRACE(0);
    const SolveItem I = A.items[it];
    const int np = I.np;
    const double* g = A.pool + I.goff;
    const int64_t ld = I.ld;
    const bool whole = I.blk == kWhole;
    const int nck = whole ? 0 : 1;
    if (whole) {
      fwd_whole(A, I, g, ld, D, stg, part, tid);
      if (A.trace && tid == 0) A.trace[8 * (size_t)it + 1] = A.trace[8 * (size_t)it + 6] = A.trace[8 * (size_t)it + 7] = gtime();
    }
    unsigned long long waited = 0;
    auto chunk_rows = [&](int, int& r0, int& nr, int& blk) {
      r0 = I.r0, nr = I.nr, blk = I.blk;
    };
    // w = b + children's contributions (children complete: the front is ready);
    // the gather of the next chunk is issued while the current one is processed
    auto gather_w = [&](int r0, int nr) {
      double v = 0.0;
      if (tid < nr) {
        const int4 src = __ldg(&A.gsrc[I.rows_off + r0 + tid]);
        if (src.x >= 0) v = A.b[src.x];
        if (src.y >= 0) v += __ldcg(&A.cbvec[src.y]);
        if (src.z >= 0) v += __ldcg(&A.cbvec[src.z]);
      }
      return v;
    };
    double wnext = 0.0;
    if (!whole) {
      int r0, nr, blk;
      chunk_rows(0, r0, nr, blk);
      wnext = gather_w(r0, nr);
    }
    for (int ck = 0; ck < nck; ++ck) {
      int r0, nr, blk;
      chunk_rows(ck, r0, nr, blk);
      if (tid < nr) wv[tid] = wnext;
      if (ck + 1 < nck) {
        int r1, nr1, b1;
        chunk_rows(ck + 1, r1, nr1, b1);
        wnext = gather_w(r1, nr1);
      }
      if (blk >= 0) load_dinv<false>(D, A.dinv + I.doff + (int64_t)kRB * kRB * blk, nr, tid);
      __syncthreads();
      if (ck == 0) RQB_TRACE(1);
      // s = L[rows, 0:ncol) y
      const int ncol = min(np, (blk >= 0 ? blk : I.npb) * kRB);
      const double* lp = g + (r0 + row);
      double s = 0.0;
      {
        // rounds: take every block published so far, stage its y, stream it;
        // the L of the first block not yet seen published is in flight during the wait
        int done = 0;
        while (done < ncol) {
          const int b1 = min(ncol, done + kRB);
          double lr[kRB / 4];
          load_block(lr, lp, ld, row < nr, done, b1, grp);
          if (tid < 32) {  // blocks published so far (counter), else poll the next block's values
            const unsigned long long w0 = A.trace ? gtime() : 0;
            int p = tid == 0 ? ld_acquire(&A.pub[I.front]) : 0;
            p = __shfl_sync(0xffffffffu, p, 0);
            int av = min(ncol, p * kRB), stgd = 0;
            if (av <= done) {
              if (!poll_block(A, A.y + I.start + done, b1 - done, stg, tid)) p = -1;
              av = b1;
              stgd = 1;
            }
            if (tid == 0) {
              avail_s = av;
              staged_s = stgd;
              if (A.trace) {
                const unsigned long long w1 = gtime();
                waited += w1 - w0;
                A.trace[8 * (size_t)it + 4] = w1;
              }
            }
          }
          __syncthreads();
          const int avail = avail_s;
          const bool stgd = staged_s;
          for (int base = done; base < avail; base += kStage) {
            const int hi = min(avail, base + kStage);
            if (!stgd)
              for (int c = tid; c < hi - base; c += kST) stg[c] = __ldcg(&A.y[I.start + base + c]);
            __syncthreads();
            if (row < nr) {
              if (base == done) {
                s += fma_block(lr, stg, b1 - done, grp);
                for (int c = b1; c < hi; c += kRB) s += block_dot(lp, ld, stg - base, c, min(hi, c + kRB), grp);
              } else {
                for (int c = base; c < hi; c += kRB) s += block_dot(lp, ld, stg - base, c, min(hi, c + kRB), grp);
              }
            }
            __syncthreads();
          }
          done = avail;
        }
      }
      part[grp][row] = s;
      if (A.trace && tid == 0) A.trace[8 * (size_t)it + 6] = gtime();
      __syncthreads();
      if (blk >= 0) {
        if (tid < 32) {
          double v0 = tid < nr ? wv[tid] - (part[0][tid] + part[1][tid] + part[2][tid] + part[3][tid]) : 0.0;
          double v1 = tid + 32 < nr
                          ? wv[tid + 32] - (part[0][tid + 32] + part[1][tid + 32] + part[2][tid + 32] + part[3][tid + 32])
                          : 0.0;
          tile_apply(D, tid, v0, v1, nr);
          if (A.trace && tid == 0) A.trace[8 * (size_t)it + 7] = gtime();
          if (tid < nr) st_relaxed(&A.y[I.start + r0 + tid], v0);
          if (tid + 32 < nr) st_relaxed(&A.y[I.start + r0 + tid + 32], v1);
        }
      } else if (tid < nr) {
        A.cbvec[I.cbvec_off + r0 + tid - np] = wv[tid] - (part[0][tid] + part[1][tid] + part[2][tid] + part[3][tid]);
      }
      __syncthreads();
    }
    RQB_TRACE(2);
    if (A.trace && tid == 0) A.trace[8 * (size_t)it + 5] = waited;
    // ---- publish; the front's last item makes the parent one step readier
    if (tid == 0) {
      if (I.blk >= 0) {
        red_release(&A.pub[I.front], 1);
        push_window(A, I.front, I.blk + A.win, I.blk + A.win);
      }
      RQB_TRACE(3);
      if (I.parent >= 0)
        item_done_fwd(A, I.parent, &keep_s);  // depth first: the parent's first item runs here next
      else
        __threadfence();
      atomicAdd(A.done, 1);
    }
  }
}

// x of one pivot row: xnew (ND order, read by descendants), caller order
// scaled, and the fused lower block of apply_operator
__device__ __forceinline__ void store_x(const SweepArgs& A, int gi, double v) {
  A.xnew[gi] = v;
  const int o = A.perm[gi];
  const double sv = A.scale * v;
  A.xout[o] = sv;
  if (A.xl_out) A.xl_out[o] = A.sigma * sv + A.vu[o];
}

// acc[q] = sum over this warp's columns c (c = warp mod 8) of U12[lane + 32 q, c] x_c:
// one warp reads whole columns (np contiguous values), 16 / kRPL columns per
// iteration, i.e. 16 loads in flight per lane
template <int kRPL>
__device__ __forceinline__ void u12_cols(const double* g, int64_t ld, int np, int ncb, const double* xc, int lane,
                                         int warp, double (&acc)[4]) {
  constexpr int kU = 16 / kRPL, kW = kST / 32;
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] = 0.0;
  const double* up = g + (int64_t)np * ld + lane;
  for (int c0 = warp; c0 < ncb; c0 += kW * kU) {
    double a[kU][kRPL];
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int q = 0; q < kRPL; ++q) {
        const int c = c0 + kW * u;
        a[u][q] = c < ncb && lane + 32 * q < np ? up[(int64_t)c * ld + 32 * q] : 0.0;
      }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int c = c0 + kW * u;
      const double xv = c < ncb ? xc[c] : 0.0;
#pragma unroll
      for (int q = 0; q < kRPL; ++q) acc[q] += a[u][q] * xv;
    }
  }
}

// L2 prefetch (one line per thread-iteration, no bulk op per column) of the
// U12 block: rows [0, np) of the columns [np, nf)
__device__ __forceinline__ void prefetch_u12(const double* g, int64_t ld, int np, int nf, int tid) {
  const int nl = (np * 8 + 127) / 128 + 1;  // lines per column (unaligned start)
  for (int i = tid; i < (nf - np) * nl; i += kST) {
    const int c = np + i / nl, l = i % nl;
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(g + (int64_t)c * ld);
    const uintptr_t a = (a0 & ~uintptr_t(127)) + 128 * l;
    if (a < a0 + 8 * np) asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
  }
}

// Backward sweep over one whole front (at most kWholeNpb pivot blocks) by one
// CTA: the ancestors' x_cb gathered at once, U12 x_cb for every pivot row
// (warp per column class, partials reduced in shared memory), then the pivot
// blocks last first: x = inv(U11) (y - U12 x_cb - U[blk, later] x_later) in warp 0.
__device__ __forceinline__ void bwd_whole(const SweepArgs& A, const SolveItem& I, const double* g, int64_t ld,
                                          const int32_t* rw, double* D, double* xs, double* pv,
                                          double (*part)[kRB], int tid) {
  constexpr int kCbBase = kWholeNpb * kRB;  // xs: [0, np) this front's x, [kCbBase, ...) x_cb
  const int np = I.np, nf = I.nf, ncb = nf - np;
  prefetch_u12(g, ld, np, nf, tid);
  if (tid == 0)  // the tile inverses, needed after the U12 product
    for (int blk = 0; blk < I.npb; ++blk) {
      const int nr = min(np, blk * kRB + kRB) - blk * kRB;
      prefetch_l2(A.dinv + I.doff + (int64_t)kRB * kRB * blk, sizeof(double) * nr * nr);
    }
  {
    constexpr int kQ = kStage / kST;
    int src[kQ];
#pragma unroll
    for (int q = 0; q < kQ; ++q) src[q] = tid + q * kST < ncb ? __ldg(&rw[np + tid + q * kST]) : -1;
#pragma unroll
    for (int q = 0; q < kQ; ++q)
      if (src[q] >= 0) xs[kCbBase + tid + q * kST] = __ldcg(&A.xnew[src[q]]);
  }
  const double yv = tid < np ? A.y[I.start + tid] : 0.0;
  __syncthreads();
  {
    const int lane = tid & 31, warp = tid >> 5;
    double acc[4];
    if (np <= 32)
      u12_cols<1>(g, ld, np, ncb, xs + kCbBase, lane, warp, acc);
    else if (np <= 64)
      u12_cols<2>(g, ld, np, ncb, xs + kCbBase, lane, warp, acc);
    else
      u12_cols<4>(g, ld, np, ncb, xs + kCbBase, lane, warp, acc);
#pragma unroll
    for (int q = 0; q < 4; ++q) D[warp * 128 + lane + 32 * q] = acc[q];  // D as scratch
    __syncthreads();
    if (tid < np) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kST / 32; ++w) s += D[w * 128 + tid];
      pv[tid] = yv - s;
    }
    __syncthreads();
  }
  const int row = tid & (kRB - 1), grp = tid >> 6;
  for (int blk = I.npb - 1; blk >= 0; --blk) {
    const int r0 = blk * kRB, nr = min(np, r0 + kRB) - r0, lo = r0 + kRB;
    load_dinv<true>(D, A.dinv + I.doff + (int64_t)kRB * kRB * blk, nr, tid);
    double s = 0.0;
    if (row < nr && lo < np) s = stream_cols(g + r0 + row, ld, xs, lo, np, grp);
    part[grp][row] = s;
    __syncthreads();
    if (tid < 32) {
      double v0 = tid < nr ? pv[r0 + tid] - (part[0][tid] + part[1][tid] + part[2][tid] + part[3][tid]) : 0.0;
      double v1 = tid + 32 < nr ? pv[r0 + tid + 32] -
                                      (part[0][tid + 32] + part[1][tid + 32] + part[2][tid + 32] + part[3][tid + 32])
                                : 0.0;
      tile_apply(D, tid, v0, v1, nr);
      if (tid < nr) {
        xs[r0 + tid] = v0;
        store_x(A, I.start + r0 + tid, v0);
      }
      if (tid + 32 < nr) {
        xs[r0 + tid + 32] = v1;
        store_x(A, I.start + r0 + tid + 32, v1);
      }
    }
    __syncthreads();
  }
}

template <int kMinBlocks>
__global__ void __launch_bounds__(kST, kMinBlocks) bwd_sweep(SweepArgs A) {
  __shared__ double D[kRB * (kRB + 1)];
  // staged x; whole-front items: [0, np) the front's own x, [kWholeNpb*64, ...) the ancestors' x_cb
  __shared__ double stg[kStage];
  __shared__ double part[4][kRB];
  __shared__ double pv[kWholeNpb * kRB];  // whole-front items: y - U12 x_cb of the pivot rows
  __shared__ int item_s, avail_s, keep_s, staged_s;
  const int tid = threadIdx.x, row = tid & (kRB - 1), grp = tid >> 6;
  if (tid == 0) keep_s = -1;
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      item_s = keep_s >= 0 ? keep_s : pop_item(A);
      keep_s = -1;
    }
    __syncthreads();
    const int it = item_s;
    if (it < 0) return;
    RQB_TRACE(0);
    const SolveItem I = A.items[it];
    const int np = I.np, nf = I.nf;
    const double* g = A.pool + I.goff;
    const int64_t ld = I.ld;
    const int32_t* rw = A.rows + I.rows_off;
    if (I.blk == kPart) {  // contribution-column chunk of one pivot block: partial sums only
      const int c0 = np + I.cbvec_off, c1 = np + I.ncbb, nr = I.nr;
      for (int c = tid; c < c1 - c0; c += kST) stg[c] = __ldcg(&A.xnew[rw[c0 + c]]);
      __syncthreads();
      double s = 0.0;
      if (row < nr) s = stream_cols(g + I.r0 + row, ld, stg - c0, c0, c1, grp);
      part[grp][row] = s;
      __syncthreads();
      if (tid < nr) A.bpart[I.ech_off + tid] = part[0][tid] + part[1][tid] + part[2][tid] + part[3][tid];
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(&A.pdone[I.front], 1);
        atomicAdd(A.done, 1);
      }
      continue;
    }
    const bool whole = I.blk == kWhole;
    if (whole) {
      bwd_whole(A, I, g, ld, rw, D, stg, pv, part, tid);
      if (A.trace && tid == 0) A.trace[8 * (size_t)it + 1] = A.trace[8 * (size_t)it + 6] = A.trace[8 * (size_t)it + 7] = gtime();
    }
    const int nck = whole ? 0 : 1;
    unsigned long long waited = 0;
    for (int ck = 0; ck < nck; ++ck) {
      const int blk = I.blk;
      const int r0 = blk * kRB, nr = min(np, r0 + kRB) - r0;
      load_dinv<true>(D, A.dinv + I.doff + (int64_t)kRB * kRB * blk, nr, tid);
      double y0 = 0.0, y1 = 0.0;
      if (tid < 32) {
        if (tid < nr) y0 = A.y[I.start + r0 + tid];
        if (tid + 32 < nr) y1 = A.y[I.start + r0 + tid + 32];
      }
      __syncthreads();
      if (ck == 0) RQB_TRACE(1);
      // columns right of this block: contribution columns (ancestors' x, final
      // since the front is ready), then this front's later pivot blocks
      const double* up = g + (r0 + row);
      const int lo = (blk + 1) * kRB;
      double s = 0.0;
      {
        for (int base = I.ncbb > 0 ? nf : np; base < nf; base += kStage) {  // chunked fronts: partial items
          const int hi = min(nf, base + kStage);
          for (int c = tid; c < hi - base; c += kST) stg[c] = __ldcg(&A.xnew[rw[base + c]]);
          __syncthreads();
          if (row < nr) s += stream_cols(up, ld, stg - base, base, hi, grp);
          __syncthreads();
        }
        // later pivot blocks are published last first: rounds over [avail_lo, done_hi);
        // the U of the next block to come is in flight during the wait
        int done_hi = np;
        while (done_hi > lo) {
          const int b0 = max(lo, ((done_hi - 1) / kRB) * kRB);
          double ur[kRB / 4];
          load_block(ur, up, ld, row < nr, b0, done_hi, grp);
          if (tid < 32) {  // blocks published so far (counter), else poll the next block's values
            const unsigned long long w0 = A.trace ? gtime() : 0;
            int p = tid == 0 ? ld_acquire(&A.pub[I.front]) : 0;
            p = __shfl_sync(0xffffffffu, p, 0);
            int av = max(lo, (I.npb - p) * kRB), stgd = 0;
            if (av >= done_hi) {
              poll_block(A, A.xnew + I.start + b0, done_hi - b0, stg, tid);
              av = b0;
              stgd = 1;
            }
            if (tid == 0) {
              avail_s = av;
              staged_s = stgd;
              if (A.trace) {
                const unsigned long long w1 = gtime();
                waited += w1 - w0;
                A.trace[8 * (size_t)it + 4] = w1;
              }
            }
          }
          __syncthreads();
          const int avail_lo = avail_s;
          const bool stgd = staged_s;
          for (int top = done_hi, bot; top > avail_lo; top = bot) {
            bot = max(avail_lo, (top - kStage + kRB - 1) / kRB * kRB);  // block aligned
            if (!stgd)
              for (int c = tid; c < top - bot; c += kST) stg[c] = __ldcg(&A.xnew[I.start + bot + c]);
            __syncthreads();
            if (row < nr) {
              if (top == done_hi) {
                s += fma_block(ur, stg + (b0 - bot), done_hi - b0, grp);
                for (int c = b0; c > bot; c -= kRB) s += block_dot(up, ld, stg - bot, c - kRB, c, grp);
              } else {
                for (int chi = top; chi > bot; chi = max(bot, (chi - 1) / kRB * kRB))
                  s += block_dot(up, ld, stg - bot, max(bot, (chi - 1) / kRB * kRB), chi, grp);
              }
            }
            __syncthreads();
          }
          done_hi = avail_lo;
        }
      }
      if (I.ncbb > 0) {  // chunked: the contribution-column partials of this block (fixed order)
        if (tid == 0) {
          unsigned long long t0 = 0;
          while (ld_acquire(&A.pdone[I.front]) < A.npart[I.front]) {
            __nanosleep(20);
            if (stalled(A, t0)) break;
          }
        }
        __syncthreads();
        if (grp == 0 && row < nr)
          for (int k = 0; k < I.ncbb; ++k) s += __ldcg(&A.bpart[I.cbvec_off + k * kRB + row]);
      }
      part[grp][row] = s;
      if (A.trace && tid == 0) A.trace[8 * (size_t)it + 6] = gtime();
      __syncthreads();
      if (tid < 32) {
        double v0 = 0.0, v1 = 0.0;
        if (tid < nr) v0 = y0 - (part[0][tid] + part[1][tid] + part[2][tid] + part[3][tid]);
        if (tid + 32 < nr)
          v1 = y1 - (part[0][tid + 32] + part[1][tid + 32] + part[2][tid + 32] + part[3][tid + 32]);
        tile_apply(D, tid, v0, v1, nr);
        if (A.trace && tid == 0) A.trace[8 * (size_t)it + 7] = gtime();
        for (int h = 0; h < 2; ++h) {
          const int r = tid + 32 * h;
          if (r < nr) {
            const double v = h ? v1 : v0;
            const int gi = I.start + r0 + r;
            st_relaxed(&A.xnew[gi], v);
            const int o = A.perm[gi];
            const double sv = A.scale * v;
            A.xout[o] = sv;
            if (A.xl_out) A.xl_out[o] = A.sigma * sv + A.vu[o];
          }
        }
      }
      __syncthreads();
    }
    RQB_TRACE(2);
    if (A.trace && tid == 0) A.trace[8 * (size_t)it + 5] = waited;
    // ---- publish; block 0 completes the front: its effective children are ready
    if (tid == 0) {
      if (!whole) {
        red_release(&A.pub[I.front], 1);
        const int v = I.npb - 1 - I.blk + A.win;
        push_window(A, I.front, v, v);
      }
      RQB_TRACE(3);
    }
    if (I.blk <= 0)  // the first effective child's first item runs here next
      for (int x = tid; x < I.nech; x += kST) front_ready(A, A.ech[I.ech_off + x], x == 0 ? &keep_s : nullptr);
    __syncthreads();
    if (tid == 0) atomicAdd(A.done, 1);
  }
}

// After factorization, one CTA per front: the net row permutation of its
// pivot block (rowperm[start + k] = pre-swap local row at position k) and the
// forward-sweep gather sources of every front row r (q = pre-swap row):
// {caller index of b (pivot rows), child-0 / child-1 contribution-vector
// entries, or -1}.
__global__ void net_rowperm(const FrontDev* __restrict__ fronts, const int32_t* __restrict__ ipiv,
                            const int32_t* __restrict__ perm, const int32_t* __restrict__ inv,
                            int32_t* __restrict__ rowperm, int4* __restrict__ gsrc) {
  // the swap sequence is replayed in shared memory (one thread; fronts above
  // kNetSmem pivots fall back to global memory)
  constexpr int kNetSmem = 4096;
  __shared__ int32_t sp[kNetSmem], sq[kNetSmem];
  const int f = blockIdx.x;
  const FrontDev F = fronts[f];
  int32_t* rp = rowperm + F.start;
  if (F.npiv <= kNetSmem) {
    for (int k = threadIdx.x; k < F.npiv; k += blockDim.x) {
      sp[k] = k;
      sq[k] = ipiv[F.start + k];
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int k = 0; k < F.npiv; ++k) {
        const int p = sq[k];
        if (p != k) {
          const int32_t t = sp[k];
          sp[k] = sp[p];
          sp[p] = t;
        }
      }
    __syncthreads();
    for (int k = threadIdx.x; k < F.npiv; k += blockDim.x) rp[k] = sp[k];
  } else if (threadIdx.x == 0) {
    for (int k = 0; k < F.npiv; ++k) rp[k] = k;
    for (int k = 0; k < F.npiv; ++k) {
      const int p = ipiv[F.start + k];
      if (p != k) {
        const int32_t t = rp[k];
        rp[k] = rp[p];
        rp[p] = t;
      }
    }
  }
  __syncthreads();
  int64_t c0off = 0, c1off = 0;
  if (F.nchild > 0) c0off = fronts[F.child0].cbvec_off - fronts[F.child0].npiv;
  if (F.nchild > 1) c1off = fronts[F.child1].cbvec_off - fronts[F.child1].npiv;
  const int32_t* inv0 = inv + F.inv_off;
  for (int r = threadIdx.x; r < F.nf; r += blockDim.x) {
    const int q = r < F.npiv ? rp[r] : r;
    int4 v;
    v.x = q < F.npiv ? perm[F.start + q] : -1;
    v.y = -1;
    v.z = -1;
    v.w = 0;
    if (F.nchild > 0) {
      const int ir = inv0[q];
      if (ir >= 0) v.y = static_cast<int>(c0off + ir);
    }
    if (F.nchild > 1) {
      const int ir = inv0[F.nf + q];
      if (ir >= 0) v.z = static_cast<int>(c1off + ir);
    }
    gsrc[F.rows_off + r] = v;
  }
}

// Inverse of every pivot block's diagonal tile after the factorization.
// Persistent CTAs take (tile, triangle) items: L11 itself (unit diagonal) and
// J U11 J (J the nr x nr reversal), both lower triangular, zero padded to
// 64 x 64 with a unit diagonal in the padding. Blocked in 32 x 32 halves:
// the diagonal halves are inverted by warps 0 / 1 (a lane owns one column in
// registers, broadcast reads, straight-line code small enough to stay in the
// instruction cache), then X21 = -X22 (M21 X11) by all four warps. The L item
// writes the strictly lower part of the tile's square, the U item the upper
// part incl. the diagonal (contiguous, column-major, ld = nr).
struct DiagBlk {
  int64_t goff;
  int32_t ld, r0, nr, doff;
};
constexpr int kInvT = 128;   // threads per CTA
constexpr int kML = kRB + 1;  // leading dimension of the tile in shared memory

__global__ void __launch_bounds__(kInvT, 4) diag_inverse(const DiagBlk* __restrict__ blks, int ntiles,
                                                      const double* __restrict__ pool, double* __restrict__ dinv) {
  __shared__ double M[kRB * kML];
  __shared__ double T[32 * 33];
  __shared__ double rd[kRB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int item = blockIdx.x; item < 2 * ntiles; item += gridDim.x) {
    const int up = item & 1;
    const DiagBlk B = blks[item >> 1];
    const int nr = B.nr;
    const bool two = nr > 32;
    const int nb = two ? kRB : 32, lnb = two ? 6 : 5;  // padded size, log2
    const double* g = pool + B.goff + B.r0 + (int64_t)B.r0 * B.ld;
    __syncthreads();  // the previous item is done with shared memory
    for (int i0 = 0; i0 < nb * nb; i0 += 16 * kInvT) {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {  // all loads in flight, then the stores
        const int idx = i0 + tid + u * kInvT, r = idx & (nb - 1), c = idx >> lnb;
        v[u] = 0.0;
        if (idx < nb * nb && r >= c) {
          if (r >= nr || c >= nr)
            v[u] = r == c ? 1.0 : 0.0;
          else if (!up)
            v[u] = r == c ? 1.0 : g[r + (int64_t)c * B.ld];
          else
            v[u] = g[(nr - 1 - r) + (int64_t)(nr - 1 - c) * B.ld];
        }
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int idx = i0 + tid + u * kInvT;
        if (idx < nb * nb) M[(idx & (nb - 1)) + (idx >> lnb) * kML] = v[u];
      }
    }
    __syncthreads();
    if (tid < nb) rd[tid] = 1.0 / M[tid + tid * kML];
    __syncthreads();
    const int o = 32 * warp;
    double x[32];
    if (warp == 0 || (warp == 1 && two)) {  // X_ww = inv(M_ww), column `lane`
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = i == lane ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        x[k] *= rd[o + k];
#pragma unroll
        for (int i = k + 1; i < 32; ++i) x[i] -= M[(o + i) + (o + k) * kML] * x[k];
      }
    }
    __syncthreads();
    if (warp == 0 || (warp == 1 && two)) {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i >= lane) M[(o + i) + (o + lane) * kML] = x[i];
    }
    __syncthreads();
    if (two) {
      // T = M21 X11 (X11 lower): thread = column lane, rows warp*8 .. +8
      double acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = 0.0;
      for (int m = lane; m < 32; ++m) {
        const double xm = M[m + lane * kML];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] += M[(32 + warp * 8 + q) + m * kML] * xm;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) T[(warp * 8 + q) + lane * 33] = acc[q];
      __syncthreads();
      // X21 = -X22 T (X22 lower), written over M21
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = 0.0;
      for (int m = 0; m < 32; ++m) {
        const double t = T[m + lane * 33];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (m <= warp * 8 + q) acc[q] += M[(32 + warp * 8 + q) + (32 + m) * kML] * t;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) M[(32 + warp * 8 + q) + lane * kML] = -acc[q];
      __syncthreads();
    }
    double* out = dinv + B.doff;
    {
      const int r = tid & (kRB - 1);
      if (r < nr)
        for (int c = tid >> 6; c < nr; c += kInvT / kRB) {
          if (!up && r > c) out[r + c * nr] = M[r + c * kML];
          if (up && r <= c) out[r + c * nr] = M[(nr - 1 - r) + (nr - 1 - c) * kML];
        }
    }
  }
}

void FactorEngine::solve_device(const double* b, double* x, double scale_out) {
  rqb_solve_enqueue(*this, b, x, scale_out, nullptr, 0.0, nullptr);
}

void FactorEngine::check_sweeps() {
  int st = 0;
  RQB_CUDA(cudaMemcpyAsync(&st, d_sweep_stall.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
  RQB_CUDA(cudaStreamSynchronize(stream));
  if (st) {
    RQB_CUDA(cudaMemsetAsync(d_sweep_stall.p, 0, sizeof(int), stream));
    fail(errc::solver, "triangular sweep stalled (watchdog): a dependency of the solve never resolved");
  }
}

void rqb_solve_prepare(FactorEngine& fe) {
  const Symbolic& S = fe.sym;
  const int nfr = static_cast<int>(S.fronts.size());
  std::vector<SolveItem> fwd, bwd;
  std::vector<int32_t> ech, fbase_f(nfr), fcnt_f(nfr), fbase_b(nfr, 0), fcnt_b(nfr, 0);
  std::vector<std::vector<int32_t>> echl(nfr);
  std::vector<int32_t> npb(nfr), ncbb(nfr);
  int64_t cbtot = 0;
  fe.win_f = std::getenv("RQB_WIN_F") ? std::max(1, std::atoi(std::getenv("RQB_WIN_F"))) : kWin;
  fe.win_b = std::getenv("RQB_WIN_B") ? std::max(1, std::atoi(std::getenv("RQB_WIN_B"))) : kWin;
  for (int f = 0; f < nfr; ++f) {
    const Front& F = S.fronts[f];
    npb[f] = (F.npiv + kRB - 1) / kRB;
    ncbb[f] = (F.nf - F.npiv + kRB - 1) / kRB;
    if (npb[f] + ncbb[f] == 0) throw Error(errc::solver, "solve: front without rows");
    if (npb[f] > 0) {
      int a = F.parent;  // nearest ancestor with pivots (empty separators pass through)
      while (a >= 0 && S.fronts[a].npiv == 0) a = S.fronts[a].parent;
      if (a >= 0) echl[a].push_back(f);
    }
    cbtot = std::max<int64_t>(cbtot, fe.fronts_h[f].cbvec_off + F.nf);
  }
  if (static_cast<int64_t>(S.rows.size()) > INT32_MAX || cbtot > INT32_MAX || fe.n > INT32_MAX)
    throw Error(errc::solver, "solve: index range exceeds int32");
  // diagonal-tile inverses: per front its pivot blocks' squares, contiguous
  std::vector<int32_t> doff_f(nfr);
  std::vector<DiagBlk> dblk;
  int64_t dtot = 0;
  for (int f = 0; f < nfr; ++f) {
    const Front& F = S.fronts[f];
    doff_f[f] = static_cast<int32_t>(dtot);
    for (int b = 0; b < npb[f]; ++b) {
      const int nr = std::min(F.npiv, (b + 1) * kRB) - b * kRB;
      dblk.push_back(DiagBlk{fe.fronts_h[f].off, fe.fronts_h[f].ld, b * kRB, nr, static_cast<int32_t>(dtot)});
      dtot += static_cast<int64_t>(nr) * nr;
      if (dtot > INT32_MAX) throw Error(errc::solver, "solve: diagonal-tile inverses exceed int32 offsets");
    }
  }
  fe.n_dblk = static_cast<int>(dblk.size());
  if (dblk.empty()) dblk.push_back(DiagBlk{});
  fe.d_dblk.upload(dblk.data(), sizeof(DiagBlk) * dblk.size(), fe.stream);
  fe.d_dinv.alloc(sizeof(double) * std::max<int64_t>(1, dtot));
  int32_t eoff = 0;
  std::vector<int32_t> ech_off(nfr);
  for (int f = 0; f < nfr; ++f) {
    ech_off[f] = eoff;
    ech.insert(ech.end(), echl[f].begin(), echl[f].end());
    eoff += static_cast<int32_t>(echl[f].size());
  }
  auto item = [&](int f, int r0, int r1, int blk) {
    const Front& F = S.fronts[f];
    const FrontDev& D = fe.fronts_h[f];
    SolveItem it{};
    it.goff = D.off;
    it.front = f;
    it.r0 = r0;
    it.nr = r1 - r0;
    it.blk = blk;
    it.ld = D.ld;
    it.np = F.npiv;
    it.nf = F.nf;
    it.start = D.start;
    it.npb = npb[f];
    it.ncbb = ncbb[f];
    it.parent = F.parent;
    it.rows_off = static_cast<int32_t>(D.rows_off);
    it.cbvec_off = static_cast<int32_t>(D.cbvec_off);
    it.ech_off = ech_off[f];
    it.nech = static_cast<int32_t>(echl[f].size());
    it.doff = doff_f[f];
    return it;
  };
  {
    // large trees are throughput bound (3 CTAs/SM, 80 registers); small ones
    // are latency bound along the tree and prefer 2 CTAs/SM without spills
    int items = 0;
    for (int f = 0; f < nfr; ++f) items += npb[f] + ncbb[f];
    fe.sweep_occ = items >= 10000 ? 3 : 2;
    if (const char* e = std::getenv("RQB_SWEEP_OCC")) fe.sweep_occ = std::atoi(e) >= 3 ? 3 : 2;
    int nsm = 148, occ = 1;
    RQB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, fe.device));
    if (fe.sweep_occ == 3)
      RQB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fwd_sweep<3>, kST, 0));
    else
      RQB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fwd_sweep<2>, kST, 0));
    fe.solve_grid = std::max(1, nsm * std::max(1, occ));
  }
  // whole-front items only on levels wide enough to keep every CTA busy
  std::vector<int> lvl_count;
  for (const Front& F : S.fronts) {
    if (F.level >= static_cast<int>(lvl_count.size())) lvl_count.resize(F.level + 1, 0);
    ++lvl_count[F.level];
  }
  // (measured: 128 fronts for small trees, 256 for large ones)
  const int whole_min = std::getenv("RQB_WHOLE_MIN") ? std::atoi(std::getenv("RQB_WHOLE_MIN"))
                                                      : (fe.sweep_occ == 3 ? 256 : 128);
  std::vector<char> whole(nfr);
  std::vector<int32_t> vnpb_f(nfr);
  for (int f = 0; f < nfr; ++f) {
    const Front& F = S.fronts[f];
    whole[f] = npb[f] <= kWholeNpb && F.nf - F.npiv <= kWholeCb && lvl_count[F.level] >= whole_min;
    vnpb_f[f] = whole[f] ? 0 : npb[f];
    fbase_f[f] = static_cast<int32_t>(fwd.size());
    if (whole[f]) {
      fwd.push_back(item(f, 0, F.nf, kWhole));
    } else {
      for (int b = 0; b < npb[f]; ++b) fwd.push_back(item(f, b * kRB, std::min(F.npiv, (b + 1) * kRB), b));
      for (int r = F.npiv; r < F.nf; r += kRB) fwd.push_back(item(f, r, std::min(F.nf, r + kRB), -1));
    }
    fcnt_f[f] = static_cast<int32_t>(fwd.size()) - fbase_f[f];
  }
  std::vector<int32_t> npart_b(nfr, 0), vnpb_b(nfr, 0);
  int64_t pslots = 0;
  // contribution-column chunk width of the backward partial items (RQB_CB_CHUNK, 64..kStage)
  const int cb_chunk = std::getenv("RQB_CB_CHUNK")
                           ? std::min(kStage, std::max(kRB, std::atoi(std::getenv("RQB_CB_CHUNK"))))
                           : kCbChunk;
  for (int f = nfr - 1; f >= 0; --f) {
    const Front& F = S.fronts[f];
    fbase_b[f] = static_cast<int32_t>(bwd.size());
    vnpb_b[f] = whole[f] ? (npb[f] > 0 ? 1 : 0) : npb[f];
    const int ncb = F.nf - F.npiv;
    if (!whole[f] && npb[f] > 0 && ncb > cb_chunk) {  // contribution-column partial items
      const int nck = (ncb + cb_chunk - 1) / cb_chunk;
      for (int b = npb[f] - 1; b >= 0; --b)
        for (int k = 0; k < nck; ++k) {
          SolveItem it = item(f, b * kRB, std::min(F.npiv, (b + 1) * kRB), kPart);
          it.cbvec_off = k * cb_chunk;
          it.ncbb = std::min(ncb, (k + 1) * cb_chunk);
          it.ech_off = static_cast<int32_t>(pslots + (static_cast<int64_t>(b) * nck + k) * kRB);
          it.nech = 0;
          it.parent = -1;
          bwd.push_back(it);
        }
      npart_b[f] = npb[f] * nck;
      for (int b = npb[f] - 1; b >= 0; --b) {
        SolveItem it = item(f, b * kRB, std::min(F.npiv, (b + 1) * kRB), b);
        it.ncbb = nck;
        it.cbvec_off = static_cast<int32_t>(pslots + static_cast<int64_t>(b) * nck * kRB);
        bwd.push_back(it);
      }
      pslots += static_cast<int64_t>(npb[f]) * nck * kRB;
      if (pslots > INT32_MAX) throw Error(errc::solver, "solve: partial-sum slots exceed int32");
      fcnt_b[f] = static_cast<int32_t>(bwd.size()) - fbase_b[f];
      continue;
    }
    if (whole[f] && npb[f] > 0) {
      bwd.push_back(item(f, 0, F.npiv, kWhole));
    } else {
      for (int b = npb[f] - 1; b >= 0; --b) {
        SolveItem it = item(f, b * kRB, std::min(F.npiv, (b + 1) * kRB), b);
        it.ncbb = 0;  // contribution columns streamed by the block item itself
        bwd.push_back(it);
      }
    }
    fcnt_b[f] = static_cast<int32_t>(bwd.size()) - fbase_b[f];
  }
  // dataflow state template: front deps (forward: children; backward: the
  // nearest ancestor with pivots), initial ready queues = the items of the
  // fronts ready at launch, in front order, counters zero
  std::vector<int32_t> dfwd(nfr), dbwd(nfr);
  std::vector<int32_t> qf(std::max<size_t>(1, fwd.size()), -1), qb(std::max<size_t>(1, bwd.size()), -1);
  int nf0 = 0, nb0 = 0;
  for (int f = 0; f < nfr; ++f) {
    const Front& F = S.fronts[f];
    dfwd[f] = 0;  // forward: items of the children still to finish
    for (int32_t c : F.children) dfwd[f] += fcnt_f[c];
    int a = F.parent;
    while (a >= 0 && S.fronts[a].npiv == 0) a = S.fronts[a].parent;
    dbwd[f] = a >= 0 ? 1 : 0;
  }
  for (int f = 0; f < nfr; ++f) {
    if (dfwd[f] == 0) {  // window: pivot blocks [0, win) (+ contribution items if npb < win)
      const int n = vnpb_f[f] < fe.win_f ? fcnt_f[f] : fe.win_f;
      for (int i = 0; i < n; ++i) qf[nf0++] = fbase_f[f] + i;
    }
    if (dbwd[f] == 0)
      for (int i = 0; i < npart_b[f] + std::min(vnpb_b[f], fe.win_b); ++i) qb[nb0++] = fbase_b[f] + i;
  }
  fe.n_fwd_items = static_cast<int>(fwd.size());
  fe.n_bwd_items = static_cast<int>(bwd.size());
  if (fwd.empty()) fwd.push_back(SolveItem{});
  if (bwd.empty()) bwd.push_back(SolveItem{});
  if (ech.empty()) ech.push_back(0);
  fe.d_items_fwd.upload(fwd.data(), sizeof(SolveItem) * fwd.size(), fe.stream);
  fe.d_items_bwd.upload(bwd.data(), sizeof(SolveItem) * bwd.size(), fe.stream);
  std::vector<int32_t> fmeta;  // fbase_f, fcnt_f, fbase_b, fcnt_b, forward window npb (0: whole front)
  fmeta.insert(fmeta.end(), fbase_f.begin(), fbase_f.end());
  fmeta.insert(fmeta.end(), fcnt_f.begin(), fcnt_f.end());
  fmeta.insert(fmeta.end(), fbase_b.begin(), fbase_b.end());
  fmeta.insert(fmeta.end(), fcnt_b.begin(), fcnt_b.end());
  fmeta.insert(fmeta.end(), vnpb_f.begin(), vnpb_f.end());
  fmeta.insert(fmeta.end(), vnpb_b.begin(), vnpb_b.end());
  fmeta.insert(fmeta.end(), npart_b.begin(), npart_b.end());
  fe.d_bpart.alloc(sizeof(double) * std::max<int64_t>(1, pslots));
  fe.d_sf.upload(fmeta.data(), sizeof(int32_t) * fmeta.size(), fe.stream);
  fe.d_ech.upload(ech.data(), sizeof(int32_t) * ech.size(), fe.stream);
  fe.d_gsrc.alloc(sizeof(int4) * std::max<size_t>(1, S.rows.size()));
  std::vector<int32_t> st;
  fe.st_dep_fwd = 0;
  st.insert(st.end(), dfwd.begin(), dfwd.end());
  fe.st_dep_bwd = static_cast<int64_t>(st.size());
  st.insert(st.end(), dbwd.begin(), dbwd.end());
  fe.st_q_fwd = static_cast<int64_t>(st.size());
  st.insert(st.end(), qf.begin(), qf.end());
  fe.st_q_bwd = static_cast<int64_t>(st.size());
  st.insert(st.end(), qb.begin(), qb.end());
  fe.st_qctl = static_cast<int64_t>(st.size());
  st.insert(st.end(), {0, nf0, 0, nb0, 0, 0});  // {head, tail} fwd, bwd; items done fwd, bwd
  fe.st_cnt = static_cast<int64_t>(st.size());  // fwd published, fwd finished, bwd published
  st.resize(st.size() + 4 * static_cast<size_t>(nfr), 0);  // + bwd partial items done
  fe.d_state0.upload(st.data(), sizeof(int32_t) * st.size(), fe.stream);
  fe.d_state.alloc(fe.d_state0.bytes);
  fe.d_rowperm.alloc(sizeof(int32_t) * std::max<int64_t>(1, fe.n));
  fe.d_sweep_stall.alloc(sizeof(int));
  RQB_CUDA(cudaMemsetAsync(fe.d_sweep_stall.p, 0, sizeof(int), fe.stream));
}

void rqb_rowperm_enqueue(FactorEngine& fe) {
  const int nfr = static_cast<int>(fe.fronts_h.size());
  net_rowperm<<<nfr, 128, 0, fe.stream>>>(fe.d_fronts.as<FrontDev>(), fe.d_ipiv.as<int32_t>(),
                                          fe.d_perm.as<int32_t>(), fe.d_inv.as<int32_t>(),
                                          fe.d_rowperm.as<int32_t>(), fe.d_gsrc.as<int4>());
  if (fe.n_dblk > 0) {
    int nsm = 148, occ = 1;
    RQB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, fe.device));
    RQB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, diag_inverse, kInvT, 0));
    const int grid = std::min(2 * fe.n_dblk, nsm * std::max(1, occ));
    diag_inverse<<<grid, kInvT, 0, fe.stream>>>(fe.d_dblk.as<DiagBlk>(), fe.n_dblk, fe.d_pool.as<double>(),
                                               fe.d_dinv.as<double>());
  }
}

void rqb_solve_enqueue(FactorEngine& fe, const double* b, double* x, double scale, const double* vu,
                       double sigma, double* xl) {
  const int nfr = static_cast<int>(fe.fronts_h.size());
  cudaStream_t st = fe.stream;
  RQB_CUDA(cudaMemcpyAsync(fe.d_state.p, fe.d_state0.p, fe.d_state0.bytes, cudaMemcpyDeviceToDevice, st));
  // published-by-value entries start unset (all-ones bit pattern, kUnset)
  RQB_CUDA(cudaMemsetAsync(fe.d_y.p, 0xff, sizeof(double) * fe.n, st));
  RQB_CUDA(cudaMemsetAsync(fe.d_xnew.p, 0xff, sizeof(double) * fe.n, st));
  int* sb = fe.d_state.as<int>();
  SweepArgs A{};
  unsigned long long* trace = nullptr;
  {
    static int traced = 0;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (std::getenv("RQB_SOLVE_TRACE") && cs == cudaStreamCaptureStatusNone && traced < 3) {
      ++traced;
      RQB_CUDA(cudaMalloc(&trace, sizeof(unsigned long long) * 8 * (size_t)(fe.n_fwd_items + fe.n_bwd_items)));
    }
  }
  A.trace = trace;
  A.ech = fe.d_ech.as<int32_t>();
  A.gsrc = fe.d_gsrc.as<int4>();
  A.stall = fe.d_sweep_stall.as<int>();
  A.pool = fe.d_pool.as<double>();
  A.dinv = fe.d_dinv.as<double>();
  A.perm = fe.d_perm.as<int32_t>();
  A.rows = fe.d_rows.as<int32_t>();
  A.b = b;
  A.y = fe.d_y.as<double>();
  A.cbvec = fe.d_cbvec.as<double>();
  A.xnew = fe.d_xnew.as<double>();
  A.xout = x;
  A.scale = scale;
  A.vu = vu;
  A.sigma = sigma;
  A.xl_out = xl;
  SweepArgs F = A;
  F.items = fe.d_items_fwd.as<SolveItem>();
  F.nitems = fe.n_fwd_items;
  F.deps = sb + fe.st_dep_fwd;
  F.queue = sb + fe.st_q_fwd;
  F.qctl = sb + fe.st_qctl;
  F.done = sb + fe.st_qctl + 4;
  F.pub = sb + fe.st_cnt;
  F.fin = sb + fe.st_cnt + nfr;
  F.fwd = 1;
  F.win = fe.win_f;
  F.fbase = fe.d_sf.as<int32_t>();
  F.fcnt = F.fbase + nfr;
  F.npb = fe.d_sf.as<int32_t>() + 4 * nfr;
  if (fe.n_fwd_items > 0) {
    if (fe.sweep_occ == 3)
      fwd_sweep<3><<<std::min(fe.solve_grid, fe.n_fwd_items), kST, 0, st>>>(F);
    else
      fwd_sweep<2><<<std::min(fe.solve_grid, fe.n_fwd_items), kST, 0, st>>>(F);
  }
  SweepArgs B = A;
  B.items = fe.d_items_bwd.as<SolveItem>();
  B.nitems = fe.n_bwd_items;
  B.deps = sb + fe.st_dep_bwd;
  B.queue = sb + fe.st_q_bwd;
  B.qctl = sb + fe.st_qctl + 2;
  B.done = sb + fe.st_qctl + 5;
  B.pub = sb + fe.st_cnt + 2 * nfr;
  B.fin = nullptr;
  B.fwd = 0;
  B.win = fe.win_b;
  B.trace = trace ? trace + 8 * (size_t)fe.n_fwd_items : nullptr;
  B.fbase = fe.d_sf.as<int32_t>() + 2 * nfr;
  B.fcnt = B.fbase + nfr;
  B.npb = fe.d_sf.as<int32_t>() + 5 * nfr;
  B.npart = fe.d_sf.as<int32_t>() + 6 * nfr;
  B.pdone = sb + fe.st_cnt + 3 * nfr;
  B.bpart = fe.d_bpart.as<double>();
  if (fe.n_bwd_items > 0) {
    if (fe.sweep_occ == 3)
      bwd_sweep<3><<<std::min(fe.solve_grid, fe.n_bwd_items), kST, 0, st>>>(B);
    else
      bwd_sweep<2><<<std::min(fe.solve_grid, fe.n_bwd_items), kST, 0, st>>>(B);
  }
  RQB_CUDA(cudaGetLastError());
  fe.launches_solve = 2;
  if (trace) {  // development trace: dump forward and backward item timings once per call
    cudaStreamSynchronize(st);
    std::vector<unsigned long long> h(8 * (size_t)(fe.n_fwd_items + fe.n_bwd_items));
    cudaMemcpy(h.data(), trace, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
    if (FILE* fp = std::fopen(std::getenv("RQB_SOLVE_TRACE"), "ab")) {
      const int32_t hdr[2] = {fe.n_fwd_items, fe.n_bwd_items};
      std::fwrite(hdr, sizeof(hdr), 1, fp);
      std::fwrite(h.data(), sizeof(unsigned long long), h.size(), fp);
      std::fclose(fp);
    }
    cudaFree(trace);
  }
}

void rqb_solve_set_attrs(int) {}

}  // namespace rqb
