// SPDX-License-Identifier: Apache-2.0
// Multi-right-hand-side forward/backward substitution over the device-resident
// fronts (solve_factored, applied to up to 8 vectors at once;
// the block Krylov-Schur reads L and U once per block of
// vectors instead of once per vector).
//
// Same dataflow skeleton as the single-vector sweeps (trisolve.cu): persistent
// CTAs claim work items from a FIFO ready queue; an item is a 64-row block of
// a front (or a whole small front); a front's items are pushed in order when
// the front becomes ready, and an item waits only on earlier items of its own
// front (published per pivot block through a release counter). The
// differences are in the data: every solution / contribution entry is a row
// of KR values (y, x and the contribution vectors are stored row-interleaved,
// [row][KR], one 32- or 64-byte segment per row), every L / U element loaded
// from HBM feeds KR multiply-adds (staged right-hand sides broadcast from
// shared memory, 8 column loads in flight per thread), and the 64x64 diagonal
// tile inverse is applied to a 64 x KR block by all 256 threads.
//
//   forward   w = b(pivot rows, caller order via the net row permutation) +
//             children's contribution rows; pivot block j: y_j = inv(L_jj)
//             (w_j - L_j,<j y_<j); contribution rows: w - L_cb,piv y -> the
//             front's contribution rows for the parent
//   backward  x_j = inv(U_jj) (y_j - U_j,>j x_>j - U_j,cb x_cb); writes x
//             (ND order, interleaved, read by descendants), the caller-order
//             result scaled, and the fused r_l = s r_u + v_u of apply_operator
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "device.cuh"

namespace rqb {

namespace {

constexpr int kMB = 64;         // rows per item
constexpr int kMT = 256;        // threads per CTA
constexpr int kMStage = 256;    // staged solution rows per round
constexpr int kMWholeNf = 512;  // whole-front items: nf bound (their y / x live in shared memory)
constexpr int kMWhole = -2;     // MItem::blk of a whole-front item
constexpr int kMPart = -3;      // MItem::blk of a backward partial item (contribution-column chunk of a block)
constexpr int kMCbChunk = 256;  // contribution columns per backward partial item
constexpr int kMSlot = kMB * 8; // doubles per partial-sum slot (64 rows x up to 8 right-hand sides)
constexpr int kDL = kMB + 1;    // leading dimension of the diagonal tile in shared memory

struct MItem {
  int64_t goff;  // front's pool offset (doubles)
  int32_t front, r0, nr, blk;  // rows [r0, r0+nr); pivot block, -1 contribution rows, kMWhole
  int32_t ld, np, nf, start;
  int32_t npb, parent, rows_off, cbvec_off;
  int32_t ech_off, nech, doff, pad;
};

struct MArgs {
  const MItem* items;
  int nitems;
  int* deps;   // per front: unfinished predecessor items (fwd) / fronts (bwd)
  int* queue;
  int* qctl;   // {head, tail}
  int* done;   // items finished (termination: items kept by a CTA never pass through the queue)
  int* pub;    // per front: pivot blocks published
  int* pdone;  // backward: per front, partial items finished
  const int32_t* npart;  // backward: per front, partial items (0: blocks stream their contribution columns)
  double* bpart;         // backward partial sums, kMSlot doubles per (front, block, chunk)
  const int32_t* fbase;
  const int32_t* fcnt;
  const int32_t* ech;  // backward: effective children (nearest descendants with pivots)
  const int4* gsrc;    // forward gather sources per front row {b, child0 cb, child1 cb, -}
  const double* pool;
  const double* dinv;
  const int32_t* perm;
  const int32_t* rows;
  const double* b;
  int64_t ldb, bsr;  // b[i * bsr + j * ldb]: column-major (bsr 1) or row-interleaved (ldb 1)
  double* y;      // [n][KR]
  double* cbvec;  // [cbvec][KR]
  double* xnew;   // [n][KR]
  double* xout;
  int64_t ldx;
  double scale;
  const double* vu;
  int64_t ldv;
  double sigma;
  double* xl;  // stride ldx
  int nrhs;
  int warp_items;        // warp items batched (RQB_MWARP=0: every item CTA-wide)
  int* blist;            // batch lists: warp items in the order they became ready (-1 unset)
  int* pcnt;             // per level: warp items that became ready
  const int32_t* bbase;  // per level: first blist entry
  const int32_t* bcnt;   // per level: warp items that become ready during the sweep (this KR)
  int* stall;
  unsigned long long* trace;  // development trace (RQB_MSOLVE_TRACE): per item start, end
};

__device__ __forceinline__ unsigned long long mtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int ld_acq(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_rel(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr unsigned long long kMStallNs = 4000000000ull;
__device__ __forceinline__ bool mstalled(const MArgs& A, unsigned long long& t0) {
  if (*((volatile int*)A.stall)) return true;
  const unsigned long long t = mtime();
  if (t0 == 0) t0 = t;
  if (t - t0 > kMStallNs) {
    atomicExch(A.stall, 1);
    return true;
  }
  return false;
}

// push the items of front f from its `from`-th on (the earlier ones are kept
// by the calling CTA: depth-first, the data it just produced is still in L2)
__device__ __forceinline__ void mpush(const MArgs& A, int f, int from = 0) {
  const int i0 = A.fbase[f] + from, n = A.fcnt[f] - from;
  if (n <= 0) return;
  const int slot = atomicAdd(&A.qctl[1], n);
  for (int i = 0; i < n; ++i) atomicExch(&A.queue[slot + i], i0 + i);
}

__device__ __forceinline__ int mpop(const MArgs& A) {
  const int h = atomicAdd(&A.qctl[0], 1);
  if (h >= A.nitems) return -1;
  int t;
  unsigned long long t0 = 0;
  while ((t = ld_acq(&A.queue[h])) == -1) {
    if (ld_acq(A.done) >= A.nitems) return -1;
    __nanosleep(32);
    if (mstalled(A, t0)) return -1;
  }
  return t;
}

// thread 0: wait until at least `need` pivot blocks of front f are published;
// returns the published count (or -1 on a stall)
__device__ __forceinline__ int wait_pub(const MArgs& A, int f, int need) {
  int p = ld_acq(&A.pub[f]);
  unsigned long long t0 = 0;
  while (p < need) {
    __nanosleep(32);
    if (mstalled(A, t0)) return -1;
    p = ld_acq(&A.pub[f]);
  }
  return p;
}

// Pivot-block solution entries are published by value: the sweep resets y and
// x to an all-ones bit pattern (a NaN no FP64 operation produces) and an item
// polls the 64 x KR entries of the block it needs directly (relaxed loads of
// relaxed stores, 8-byte single-copy atomic), so the chain of pivot blocks
// has no fence + counter round trip.
constexpr long long kUnsetBits = -1LL;
__device__ __forceinline__ void st_rlx(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_rlx(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// warp 0: wait until the nv (<= 64 KR) entries at src are all published, copy
// them to dst (shared memory). false if the watchdog fired.
template <int KR>
__device__ __forceinline__ bool poll_vals(const MArgs& A, const double* src, int nv, double* dst, int lane) {
  constexpr int kPer = 2 * KR;  // 64 KR / 32 lanes
  unsigned long long t0 = 0;
  for (;;) {
    double v[kPer];
    bool ok = true;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int i = lane + 32 * u;
      v[u] = i < nv ? ld_rlx(src + i) : 0.0;
      ok = ok && (i >= nv || __double_as_longlong(v[u]) != kUnsetBits);
    }
    if (__all_sync(0xffffffffu, ok)) {
#pragma unroll
      for (int u = 0; u < kPer; ++u)
        if (lane + 32 * u < nv) dst[lane + 32 * u] = v[u];
      return true;
    }
    int st = 0;
    if (lane == 0) {
      __nanosleep(20);
      st = mstalled(A, t0);
    }
    if (__shfl_sync(0xffffffffu, st, 0)) return false;
  }
}

// acc[j] += sum over the pivot-block columns [c_lo, c_hi) of this front of
// A[row, c] v[c][j], consuming one 64-column block at a time in chain order
// (ascending for the forward sweep, descending for the backward one): the
// block's matrix columns are loaded into registers before its entries are
// polled (the next block's while the current one is consumed), warp 0 polls
// and stages the block's published entries, and each block's partial is added
// to acc in block order (bitwise deterministic whatever the timing).
template <int KR, bool kAsc>
__device__ __forceinline__ void consume_blocks(const MArgs& A, const double* vals, const double* lp, int64_t ld,
                                               bool rowok, int c_lo, int c_hi, double* stg, int tid, int grp,
                                               double (&acc)[KR]) {
  if (c_lo >= c_hi) return;
  const int lane = tid & 31, warp = tid >> 5;
  auto bounds = [&](int i, int& b0, int& b1) {  // i-th block in chain order
    if (kAsc) {
      b0 = c_lo + i * kMB;
      b1 = min(c_hi, b0 + kMB);
    } else {
      const int top0 = c_lo + ((c_hi - 1 - c_lo) / kMB) * kMB;  // first (highest) block start
      b0 = top0 - i * kMB;
      b1 = min(c_hi, b0 + kMB);
    }
  };
  const int nblk = (c_hi - c_lo + kMB - 1) / kMB;
  constexpr int kU = kMB / 4;
  // KR = 8 (128 registers): the next block's columns are loaded while the
  // current one is consumed; KR = 4 (80 registers, 3 CTAs / SM): each block's
  // columns are issued right before its entries are polled
  constexpr bool kNext = KR == 8;
  double cur[kU], nxt[kNext ? kU : 1];
  int b0, b1;
  bounds(0, b0, b1);
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int c = b0 + grp + 4 * u;
    cur[u] = (rowok && c < b1) ? lp[(int64_t)c * ld] : 0.0;
  }
  for (int i = 0; i < nblk; ++i) {
    bounds(i, b0, b1);
    if (!kNext && i > 0) {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int c = b0 + grp + 4 * u;
        cur[u] = (rowok && c < b1) ? lp[(int64_t)c * ld] : 0.0;
      }
    }
    if (kNext && i + 1 < nblk) {
      int n0, n1;
      bounds(i + 1, n0, n1);
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int c = n0 + grp + 4 * u;
        nxt[kNext ? u : 0] = (rowok && c < n1) ? lp[(int64_t)c * ld] : 0.0;
      }
    }
    if (warp == 0) poll_vals<KR>(A, vals + (int64_t)b0 * KR, (b1 - b0) * KR, stg, lane);
    __syncthreads();
    double t[KR];
#pragma unroll
    for (int j = 0; j < KR; ++j) t[j] = 0.0;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int c = grp + 4 * u;
      if (c < b1 - b0) {
        const double2* xp = reinterpret_cast<const double2*>(stg + c * KR);
#pragma unroll
        for (int q = 0; q < KR / 2; ++q) {
          const double2 x = xp[q];
          t[2 * q] += cur[u] * x.x;
          t[2 * q + 1] += cur[u] * x.y;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < KR; ++j) acc[j] += t[j];
    __syncthreads();
    if (kNext)
#pragma unroll
      for (int u = 0; u < kU; ++u) cur[u] = nxt[kNext ? u : 0];
  }
}

// acc[j] += sum over this thread's column class (c = cb + grp mod 4) of
// A[row, c] xs[c][j]: eight column loads in flight per iteration, the staged
// right-hand sides read as double2 broadcasts (every lane of a warp reads the
// same column)
template <int KR>
__device__ __forceinline__ void mstream(const double* lp, int64_t ld, bool rowok, const double* xs, int cb, int ce,
                                        int grp, double (&acc)[KR]) {
  int c = cb + grp;
  for (; c + 28 < ce; c += 32) {
    double a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = rowok ? lp[(int64_t)(c + 4 * u) * ld] : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double2* xp = reinterpret_cast<const double2*>(xs + (c + 4 * u) * KR);
#pragma unroll
      for (int q = 0; q < KR / 2; ++q) {
        const double2 t = xp[q];
        acc[2 * q] += a[u] * t.x;
        acc[2 * q + 1] += a[u] * t.y;
      }
    }
  }
  if (c < ce) {
    double a[7];
#pragma unroll
    for (int u = 0; u < 7; ++u) a[u] = (rowok && c + 4 * u < ce) ? lp[(int64_t)(c + 4 * u) * ld] : 0.0;
#pragma unroll
    for (int u = 0; u < 7; ++u)
      if (c + 4 * u < ce) {
        const double2* xp = reinterpret_cast<const double2*>(xs + (c + 4 * u) * KR);
#pragma unroll
        for (int q = 0; q < KR / 2; ++q) {
          const double2 t = xp[q];
          acc[2 * q] += a[u] * t.x;
          acc[2 * q + 1] += a[u] * t.y;
        }
      }
  }
}

// diagonal tile inverse (forward: unit-lower inv(L11); backward: inv(U11)),
// zero padded to 64 x 64, into D (leading dimension kDL)
template <bool kUpper>
__device__ __forceinline__ void mload_dinv(double* D, const double* src, int nr, int tid) {
  constexpr int kPer = kMB * kMB / kMT;
  double v[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int idx = tid + u * kMT, r = idx & (kMB - 1), c = idx >> 6;
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
    const int idx = tid + u * kMT;
    D[(idx & (kMB - 1)) + (idx >> 6) * kDL] = v[u];
  }
}

// per-thread partials acc (row, grp) -> part[grp][row][KR]
template <int KR>
__device__ __forceinline__ void put_part(double* part, int grp, int row, const double (&acc)[KR]) {
  double2* p = reinterpret_cast<double2*>(part + ((grp * kMB) + row) * KR);
#pragma unroll
  for (int q = 0; q < KR / 2; ++q) p[q] = make_double2(acc[2 * q], acc[2 * q + 1]);
}

// w[r][j] -= sum_g part[g][r][j] for the nr rows (all threads)
template <int KR>
__device__ __forceinline__ void sub_parts(double* w, const double* part, int nr, int tid) {
  for (int idx = tid; idx < nr * KR; idx += kMT) {
    const int r = idx / KR, j = idx % KR;
    w[idx] -= (part[(0 * kMB + r) * KR + j] + part[(1 * kMB + r) * KR + j]) +
              (part[(2 * kMB + r) * KR + j] + part[(3 * kMB + r) * KR + j]);
  }
}

// out[j] = sum_c D[row, c] w[c][j] for this thread's columns j = jq * KR/4 + t
template <int KR>
__device__ __forceinline__ void tile_mul(const double* D, const double* w, int nr, int row, int jq,
                                         double (&out)[KR / 4]) {
  constexpr int kJ = KR / 4;
#pragma unroll
  for (int t = 0; t < kJ; ++t) out[t] = 0.0;
  for (int c = 0; c < nr; ++c) {
    const double d = D[row + c * kDL];
#pragma unroll
    for (int t = 0; t < kJ; ++t) out[t] += d * w[c * KR + jq * kJ + t];
  }
}

// w rows [r0, r0 + nr) of the front: b (pivot rows) + children's contribution rows
template <int KR>
__device__ __forceinline__ void gather_w(const MArgs& A, const MItem& I, int r0, int nr, double* w, int tid) {
  for (int idx = tid; idx < nr * KR; idx += kMT) {
    const int r = idx / KR, j = idx % KR;
    const int4 src = __ldg(&A.gsrc[I.rows_off + r0 + r]);
    double v = 0.0;
    if (src.x >= 0 && j < A.nrhs) v = A.b[src.x * A.bsr + j * A.ldb];
    if (src.y >= 0) v += __ldcg(&A.cbvec[(int64_t)src.y * KR + j]);
    if (src.z >= 0) v += __ldcg(&A.cbvec[(int64_t)src.z * KR + j]);
    w[idx] = v;
  }
}

template <int KR>
struct MSmem {
  double* D;     // 64 x kDL
  double* part;  // 4 x 64 x KR
  double* w;     // 64 x KR
  double* stg;   // max(kMStage, kMWholeNf) x KR
};

template <int KR>
__device__ __forceinline__ MSmem<KR> carve(double* sm) {
  MSmem<KR> s;
  s.D = sm;
  s.part = s.D + kMB * kDL;
  s.w = s.part + 4 * kMB * KR;
  s.stg = s.w + kMB * KR;
  return s;
}

template <int KR>
constexpr size_t msmem_bytes() {
  return sizeof(double) * (kMB * kDL + 4 * kMB * KR + kMB * KR + (kMStage > kMWholeNf ? kMStage : kMWholeNf) * KR);
}

// Warp items: whole-front items of the bottom levels with one pivot block
// (npiv <= 64) and nf <= mwarp_nf<KR>() (MItem::pad == 1) are taken up to 8
// at a time by one CTA, one front per warp, each warp in its own slice of the
// CTA's shared memory with no CTA barrier: the bottom of the tree is a
// throughput phase of thousands of independent 25-100 KB fronts whose
// CTA-wide items were bound by their chain of dependent round trips (one item
// in flight per CTA); eight per CTA keep eight chains in flight.
template <int KR>
constexpr int mwarp_doubles() {
  return static_cast<int>(msmem_bytes<KR>() / sizeof(double) / (kMT / 32)) & ~1;
}
template <int KR>
constexpr int mwarp_nf() {
  return mwarp_doubles<KR>() / KR;
}
template <int KR>
__device__ __forceinline__ bool mwarp_ok(const MItem& I) {  // MItem::pad: bit 0 fits KR <= 8, bit 1 KR = 4; level << 8
  return I.blk == kMWhole && (I.pad & (KR == 4 ? 2 : 1)) != 0;
}

// A queue entry v <= -2 is a batch of warp items: blist[b0 .. b0 + cnt),
// v = -2 - (8 b0 + cnt - 1). Batches are formed on the push side: a warp item
// that becomes ready takes the next entry of its level's batch list; whoever
// takes the 8th (or the level's last) entry pushes the batch once the earlier
// entries are written (their writers already hold them), so a popped batch is
// all ready items and never waits.
__device__ __forceinline__ int mbatch_entry(int b0, int cnt) { return -2 - (8 * b0 + cnt - 1); }

template <int KR>
__device__ __forceinline__ void mpush_warp(const MArgs& A, int it, int level) {
  const int base = A.bbase[level], total = A.bcnt[level];
  const int i = atomicAdd(&A.pcnt[level], 1);
  __threadfence();
  atomicExch(&A.blist[base + i], it);
  if ((i & 7) == 7 || i + 1 == total) {
    const int s0 = i & ~7;
    unsigned long long t0 = 0;
    for (int j = s0; j < i; ++j)
      while (ld_acq(&A.blist[base + j]) == -1)
        if (mstalled(A, t0)) return;
    __threadfence();
    const int slot = atomicAdd(&A.qctl[1], 1);
    atomicExch(&A.queue[slot], mbatch_entry(base + s0, i - s0 + 1));
  }
}

// push front f's items, or f's warp item into its level's batch list
template <int KR>
__device__ __forceinline__ void mpush_any(const MArgs& A, int f, int from = 0) {
  const int it = A.fbase[f];
  if (A.warp_items && A.fcnt[f] == 1) {
    const MItem& I = A.items[it];
    if (mwarp_ok<KR>(I)) {
      mpush_warp<KR>(A, it, I.pad >> 8);
      return;
    }
  }
  mpush(A, f, from);
}

// thread 0: decode a popped queue entry into batch_s (count) or -1 (single item)
__device__ __forceinline__ int mdecode(const MArgs& A, int v, int* batch) {
  if (v > -2) return 0;
  const int code = -2 - v, b0 = code >> 3, cnt = (code & 7) + 1;
  for (int w = 0; w < cnt; ++w) batch[w] = __ldcg(&A.blist[b0 + w]);
  return cnt;
}

// forward warp item: w = b + children's contribution rows (wy, nf x KR);
// y = inv(L11) w over the np <= 64 pivot rows (rows lane, lane + 32); the
// contribution rows w - L21 y (two 32-row chunks at a time) -> the front's
// contribution rows for the parent; then the parent's dependency count.
template <int KR>
__device__ void mfwd_warp(const MArgs& A, const MItem& I, double* wy, int lane) {
  const int np = I.np, nf = I.nf;
  const double* g = A.pool + I.goff;
  const int64_t ld = I.ld;
  for (int r = lane; r < nf; r += 32) {
    const int4 src = __ldg(&A.gsrc[I.rows_off + r]);
    double v[KR];
#pragma unroll
    for (int j = 0; j < KR; ++j) v[j] = (src.x >= 0 && j < A.nrhs) ? A.b[src.x * A.bsr + j * A.ldb] : 0.0;
    if (src.y >= 0)
#pragma unroll
      for (int j = 0; j < KR; ++j) v[j] += __ldcg(&A.cbvec[(int64_t)src.y * KR + j]);
    if (src.z >= 0)
#pragma unroll
      for (int j = 0; j < KR; ++j) v[j] += __ldcg(&A.cbvec[(int64_t)src.z * KR + j]);
#pragma unroll
    for (int j = 0; j < KR; ++j) wy[r * KR + j] = v[j];
  }
  __syncwarp();
  const double* D = A.dinv + I.doff;  // np x np: strictly lower inv(L11), unit diagonal
  const int r0 = lane, r1 = lane + 32;
  double o0[KR], o1[KR];
#pragma unroll
  for (int j = 0; j < KR; ++j) o0[j] = o1[j] = 0.0;
#pragma unroll 8
  for (int c = 0; c < np; ++c) {
    const double d0 = (r0 < np && c < r0) ? __ldg(&D[r0 + c * np]) : (c == r0 ? 1.0 : 0.0);
    const double d1 = (r1 < np && c < r1) ? __ldg(&D[r1 + c * np]) : (c == r1 ? 1.0 : 0.0);
    const double2* wp = reinterpret_cast<const double2*>(wy + c * KR);
#pragma unroll
    for (int q = 0; q < KR / 2; ++q) {
      const double2 x = wp[q];
      o0[2 * q] += d0 * x.x;
      o0[2 * q + 1] += d0 * x.y;
      o1[2 * q] += d1 * x.x;
      o1[2 * q + 1] += d1 * x.y;
    }
  }
  __syncwarp();  // every lane read w's pivot rows before they become y
#pragma unroll
  for (int j = 0; j < KR; ++j) {
    if (r0 < np) {
      wy[r0 * KR + j] = o0[j];
      A.y[(int64_t)(I.start + r0) * KR + j] = o0[j];
    }
    if (r1 < np) {
      wy[r1 * KR + j] = o1[j];
      A.y[(int64_t)(I.start + r1) * KR + j] = o1[j];
    }
  }
  __syncwarp();
  for (int rb = np; rb < nf; rb += 64) {
    const int ra = rb + lane, rc = rb + 32 + lane;
    const bool oka = ra < nf, okc = rc < nf;
    double a0[KR], a1[KR];
#pragma unroll
    for (int j = 0; j < KR; ++j) a0[j] = a1[j] = 0.0;
#pragma unroll 8
    for (int c = 0; c < np; ++c) {
      const double la = oka ? g[ra + (int64_t)c * ld] : 0.0;
      const double lc = okc ? g[rc + (int64_t)c * ld] : 0.0;
      const double2* yp = reinterpret_cast<const double2*>(wy + c * KR);
#pragma unroll
      for (int q = 0; q < KR / 2; ++q) {
        const double2 x = yp[q];
        a0[2 * q] += la * x.x;
        a0[2 * q + 1] += la * x.y;
        a1[2 * q] += lc * x.x;
        a1[2 * q + 1] += lc * x.y;
      }
    }
#pragma unroll
    for (int j = 0; j < KR; ++j) {
      if (oka) A.cbvec[(int64_t)(I.cbvec_off + ra - np) * KR + j] = wy[ra * KR + j] - a0[j];
      if (okc) A.cbvec[(int64_t)(I.cbvec_off + rc - np) * KR + j] = wy[rc * KR + j] - a1[j];
    }
  }
  __threadfence();
  __syncwarp();
  if (lane == 0) {
    if (I.parent >= 0) {
      int old;
      asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], -1;" : "=r"(old) : "l"(A.deps + I.parent) : "memory");
      if (old == 1) {
        __threadfence();
        mpush_any<KR>(A, I.parent);
      }
    }
    atomicAdd(A.done, 1);
  }
}

// ---------------------------------------------------------------------------
// forward sweep
template <int KR>
__device__ void mfwd_whole(const MArgs& A, const MItem& I, MSmem<KR>& S, int tid) {
  const int np = I.np, nf = I.nf, row = tid & (kMB - 1), grp = tid >> 6, jq = tid >> 6;
  const double* g = A.pool + I.goff;
  const int64_t ld = I.ld;
  double* wy = S.stg;  // [nf][KR]: w, then y over the pivot rows
  gather_w<KR>(A, I, 0, nf, wy, tid);
  const int npb = (np + kMB - 1) / kMB;
  for (int blk = 0; blk < npb; ++blk) {
    const int r0 = blk * kMB, nr = min(np, r0 + kMB) - r0;
    mload_dinv<false>(S.D, A.dinv + I.doff + (int64_t)kMB * kMB * blk, nr, tid);
    __syncthreads();  // wy complete (gather / previous block)
    double acc[KR];
#pragma unroll
    for (int j = 0; j < KR; ++j) acc[j] = 0.0;
    if (r0 > 0) mstream<KR>(g + r0 + row, ld, row < nr, wy, 0, r0, grp, acc);
    put_part<KR>(S.part, grp, row, acc);
    __syncthreads();
    sub_parts<KR>(wy + r0 * KR, S.part, nr, tid);
    __syncthreads();
    double out[KR / 4];
    tile_mul<KR>(S.D, wy + r0 * KR, nr, row, jq, out);
    __syncthreads();  // every thread read wy's block before it is overwritten
    if (row < nr)
#pragma unroll
      for (int t = 0; t < KR / 4; ++t) {
        const int j = jq * (KR / 4) + t;
        wy[(r0 + row) * KR + j] = out[t];
        A.y[(int64_t)(I.start + r0 + row) * KR + j] = out[t];
      }
  }
  __syncthreads();
  for (int r0 = np; r0 < nf; r0 += kMB) {
    const int nr = min(nf, r0 + kMB) - r0;
    double acc[KR];
#pragma unroll
    for (int j = 0; j < KR; ++j) acc[j] = 0.0;
    if (np > 0) mstream<KR>(g + r0 + row, ld, row < nr, wy, 0, np, grp, acc);
    put_part<KR>(S.part, grp, row, acc);
    __syncthreads();
    for (int idx = tid; idx < nr * KR; idx += kMT) {
      const int r = idx / KR, j = idx % KR;
      const double s = (S.part[(0 * kMB + r) * KR + j] + S.part[(1 * kMB + r) * KR + j]) +
                       (S.part[(2 * kMB + r) * KR + j] + S.part[(3 * kMB + r) * KR + j]);
      A.cbvec[(int64_t)(I.cbvec_off + r0 + r - np) * KR + j] = wy[(r0 + r) * KR + j] - s;
    }
    __syncthreads();
  }
}

template <int KR, int kMinBlocks>
__global__ void __launch_bounds__(kMT, kMinBlocks) mfwd_sweep(MArgs A) {
  extern __shared__ __align__(16) double msm[];
  MSmem<KR> S = carve<KR>(msm);
  __shared__ int item_s, keep_s, nb_s;
  __shared__ int batch_s[kMT / 32];
  const int tid = threadIdx.x, row = tid & (kMB - 1), grp = tid >> 6, jq = tid >> 6;
  if (tid == 0) keep_s = -1;
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      item_s = keep_s >= 0 ? keep_s : mpop(A);
      keep_s = -1;
      nb_s = mdecode(A, item_s, batch_s);
    }
    __syncthreads();
    const int it = item_s;
    if (it == -1) return;
    if (nb_s > 0) {  // one warp item per warp
      const int w = tid >> 5, lane = tid & 31;
      if (w < nb_s) {
        const int wi = batch_s[w];
        if (A.trace && lane == 0) A.trace[2 * (size_t)wi] = mtime();
        mfwd_warp<KR>(A, A.items[wi], msm + w * mwarp_doubles<KR>(), lane);
        if (A.trace && lane == 0) A.trace[2 * (size_t)wi + 1] = mtime();
      }
      continue;
    }
    const MItem I = A.items[it];
    if (A.trace && tid == 0) A.trace[2 * (size_t)it] = mtime();
    if (I.blk == kMWhole) {
      mfwd_whole<KR>(A, I, S, tid);
    } else {
      const double* g = A.pool + I.goff;
      const int64_t ld = I.ld;
      const int nr = I.nr, blk = I.blk, np = I.np;
      gather_w<KR>(A, I, I.r0, nr, S.w, tid);
      if (blk >= 0) mload_dinv<false>(S.D, A.dinv + I.doff + (int64_t)kMB * kMB * blk, nr, tid);
      const int ncol = blk >= 0 ? blk * kMB : np;  // y columns this item needs
      double acc[KR];
#pragma unroll
      for (int j = 0; j < KR; ++j) acc[j] = 0.0;
      __syncthreads();  // w and D staged
      consume_blocks<KR, true>(A, A.y + (int64_t)I.start * KR, g + I.r0 + row, ld, row < nr, 0, ncol, S.stg, tid,
                               grp, acc);
      put_part<KR>(S.part, grp, row, acc);
      __syncthreads();
      if (blk >= 0) {
        sub_parts<KR>(S.w, S.part, nr, tid);
        __syncthreads();
        double out[KR / 4];
        tile_mul<KR>(S.D, S.w, nr, row, jq, out);
        if (row < nr)
#pragma unroll
          for (int t = 0; t < KR / 4; ++t)
            st_rlx(&A.y[(int64_t)(I.start + I.r0 + row) * KR + jq * (KR / 4) + t], out[t]);
      } else {
        for (int idx = tid; idx < nr * KR; idx += kMT) {
          const int r = idx / KR, j = idx % KR;
          const double s = (S.part[(0 * kMB + r) * KR + j] + S.part[(1 * kMB + r) * KR + j]) +
                           (S.part[(2 * kMB + r) * KR + j] + S.part[(3 * kMB + r) * KR + j]);
          A.cbvec[(int64_t)(I.cbvec_off + I.r0 + r - np) * KR + j] = S.w[idx] - s;
        }
      }
    }
    __syncthreads();  // every row written before thread 0 releases the parent
    if (A.trace && tid == 0) A.trace[2 * (size_t)it + 1] = mtime();
    if (tid == 0) {
      if (I.parent >= 0) {
        int old;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], -1;" : "=r"(old) : "l"(A.deps + I.parent) : "memory");
        if (old == 1) {  // depth first: the parent's first item runs here next
          __threadfence();
          if (A.warp_items && A.fcnt[I.parent] == 1 && mwarp_ok<KR>(A.items[A.fbase[I.parent]])) {
            mpush_any<KR>(A, I.parent);
          } else {
            mpush(A, I.parent, 1);
            keep_s = A.fbase[I.parent];
          }
        }
      }
      atomicAdd(A.done, 1);
    }
  }
}

// ---------------------------------------------------------------------------
// backward sweep
template <int KR>
__device__ __forceinline__ void store_xm(const MArgs& A, int gi, int j, double v) {
  st_rlx(&A.xnew[(int64_t)gi * KR + j], v);
  if (j < A.nrhs) {
    const int64_t o = A.perm[gi];
    const double sv = A.scale * v;
    A.xout[o + j * A.ldx] = sv;
    if (A.xl) A.xl[o + j * A.ldx] = A.sigma * sv + A.vu[o + j * A.ldv];
  }
}

template <int KR>
__device__ void mbwd_whole(const MArgs& A, const MItem& I, MSmem<KR>& S, int tid) {
  const int np = I.np, nf = I.nf, row = tid & (kMB - 1), grp = tid >> 6, jq = tid >> 6;
  const double* g = A.pool + I.goff;
  const int64_t ld = I.ld;
  const int32_t* rw = A.rows + I.rows_off;
  double* xs = S.stg;  // [nf][KR]: x of the pivot rows (as solved), x_cb of the ancestors
  for (int idx = tid; idx < (nf - np) * KR; idx += kMT) {
    const int c = np + idx / KR, j = idx % KR;
    xs[c * KR + j] = __ldcg(&A.xnew[(int64_t)rw[c] * KR + j]);
  }
  const int npb = (np + kMB - 1) / kMB;
  for (int blk = npb - 1; blk >= 0; --blk) {
    const int r0 = blk * kMB, nr = min(np, r0 + kMB) - r0;
    mload_dinv<true>(S.D, A.dinv + I.doff + (int64_t)kMB * kMB * blk, nr, tid);
    for (int idx = tid; idx < nr * KR; idx += kMT) S.w[idx] = A.y[(int64_t)(I.start + r0) * KR + idx];
    __syncthreads();
    double acc[KR];
#pragma unroll
    for (int j = 0; j < KR; ++j) acc[j] = 0.0;
    mstream<KR>(g + r0 + row, ld, row < nr, xs, r0 + nr, nf, grp, acc);
    put_part<KR>(S.part, grp, row, acc);
    __syncthreads();
    sub_parts<KR>(S.w, S.part, nr, tid);
    __syncthreads();
    double out[KR / 4];
    tile_mul<KR>(S.D, S.w, nr, row, jq, out);
    if (row < nr)
#pragma unroll
      for (int t = 0; t < KR / 4; ++t) {
        const int j = jq * (KR / 4) + t;
        xs[(r0 + row) * KR + j] = out[t];
        store_xm<KR>(A, I.start + r0 + row, j, out[t]);
      }
    __syncthreads();
  }
}

// backward warp item (see mfwd_warp): xs[c] = the ancestors' x of the
// contribution columns c >= np; w = y - U12 x_cb over the pivot rows (rows
// lane, lane + 32, kept in xs[0, np)); x = inv(U11) w; then the effective
// children's dependency counts.
template <int KR>
__device__ void mbwd_warp(const MArgs& A, const MItem& I, double* xs, int lane) {
  const int np = I.np, nf = I.nf;
  const double* g = A.pool + I.goff;
  const int64_t ld = I.ld;
  const int32_t* rw = A.rows + I.rows_off;
  for (int idx = lane; idx < (nf - np) * KR; idx += 32) {
    const int c = np + idx / KR, j = idx % KR;
    xs[c * KR + j] = __ldcg(&A.xnew[(int64_t)rw[c] * KR + j]);
  }
  __syncwarp();
  const int r0 = lane, r1 = lane + 32;
  const bool ok0 = r0 < np, ok1 = r1 < np;
  double a0[KR], a1[KR];
#pragma unroll
  for (int j = 0; j < KR; ++j) a0[j] = a1[j] = 0.0;
#pragma unroll 8
  for (int c = np; c < nf; ++c) {
    const double u0 = ok0 ? g[r0 + (int64_t)c * ld] : 0.0;
    const double u1 = ok1 ? g[r1 + (int64_t)c * ld] : 0.0;
    const double2* xp = reinterpret_cast<const double2*>(xs + c * KR);
#pragma unroll
    for (int q = 0; q < KR / 2; ++q) {
      const double2 x = xp[q];
      a0[2 * q] += u0 * x.x;
      a0[2 * q + 1] += u0 * x.y;
      a1[2 * q] += u1 * x.x;
      a1[2 * q + 1] += u1 * x.y;
    }
  }
#pragma unroll
  for (int j = 0; j < KR; ++j) {
    if (ok0) xs[r0 * KR + j] = A.y[(int64_t)(I.start + r0) * KR + j] - a0[j];
    if (ok1) xs[r1 * KR + j] = A.y[(int64_t)(I.start + r1) * KR + j] - a1[j];
  }
  __syncwarp();
  const double* D = A.dinv + I.doff;  // np x np: upper inv(U11) (r <= c)
  double o0[KR], o1[KR];
#pragma unroll
  for (int j = 0; j < KR; ++j) o0[j] = o1[j] = 0.0;
#pragma unroll 8
  for (int c = 0; c < np; ++c) {
    const double d0 = (ok0 && r0 <= c) ? __ldg(&D[r0 + c * np]) : 0.0;
    const double d1 = (ok1 && r1 <= c) ? __ldg(&D[r1 + c * np]) : 0.0;
    const double2* wp = reinterpret_cast<const double2*>(xs + c * KR);
#pragma unroll
    for (int q = 0; q < KR / 2; ++q) {
      const double2 x = wp[q];
      o0[2 * q] += d0 * x.x;
      o0[2 * q + 1] += d0 * x.y;
      o1[2 * q] += d1 * x.x;
      o1[2 * q + 1] += d1 * x.y;
    }
  }
#pragma unroll
  for (int j = 0; j < KR; ++j) {
    if (ok0) store_xm<KR>(A, I.start + r0, j, o0[j]);
    if (ok1) store_xm<KR>(A, I.start + r1, j, o1[j]);
  }
  __threadfence();
  __syncwarp();
  for (int x = lane; x < I.nech; x += 32) {
    const int f = A.ech[I.ech_off + x];
    if (atomicSub(&A.deps[f], 1) == 1) {
      __threadfence();
      mpush_any<KR>(A, f);
    }
  }
  if (lane == 0) atomicAdd(A.done, 1);
}

template <int KR, int kMinBlocks>
__global__ void __launch_bounds__(kMT, kMinBlocks) mbwd_sweep(MArgs A) {
  extern __shared__ __align__(16) double msm[];
  MSmem<KR> S = carve<KR>(msm);
  __shared__ int item_s, keep_s, nb_s;
  __shared__ int batch_s[kMT / 32];
  const int tid = threadIdx.x, row = tid & (kMB - 1), grp = tid >> 6, jq = tid >> 6;
  if (tid == 0) keep_s = -1;
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      item_s = keep_s >= 0 ? keep_s : mpop(A);
      keep_s = -1;
      nb_s = mdecode(A, item_s, batch_s);
    }
    __syncthreads();
    const int it = item_s;
    if (it == -1) return;
    if (nb_s > 0) {  // one warp item per warp
      const int w = tid >> 5, lane = tid & 31;
      if (w < nb_s) {
        const int wi = batch_s[w];
        if (A.trace && lane == 0) A.trace[2 * (size_t)wi] = mtime();
        mbwd_warp<KR>(A, A.items[wi], msm + w * mwarp_doubles<KR>(), lane);
        if (A.trace && lane == 0) A.trace[2 * (size_t)wi + 1] = mtime();
      }
      continue;
    }
    const MItem I = A.items[it];
    if (A.trace && tid == 0) A.trace[2 * (size_t)it] = mtime();
    if (I.blk == kMPart) {
      // one contribution-column chunk [np + ech_off, np + nech) of one pivot
      // block: U[blk rows, chunk] x_chunk into its partial-sum slot, no waits
      const double* g = A.pool + I.goff;
      const int32_t* rw = A.rows + I.rows_off;
      const int c0 = I.np + I.ech_off, c1 = I.np + I.nech, nr = I.nr;
      for (int idx = tid; idx < (c1 - c0) * KR; idx += kMT) {
        const int c = c0 + idx / KR, j = idx % KR;
        S.stg[idx] = __ldcg(&A.xnew[(int64_t)rw[c] * KR + j]);
      }
      double acc[KR];
#pragma unroll
      for (int j = 0; j < KR; ++j) acc[j] = 0.0;
      __syncthreads();
      mstream<KR>(g + I.r0 + row, I.ld, row < nr, S.stg - c0 * KR, c0, c1, grp, acc);
      put_part<KR>(S.part, grp, row, acc);
      __syncthreads();
      for (int idx = tid; idx < nr * KR; idx += kMT) {
        const int r = idx / KR, j = idx % KR;
        A.bpart[(int64_t)I.cbvec_off + idx] = (S.part[(0 * kMB + r) * KR + j] + S.part[(1 * kMB + r) * KR + j]) +
                                              (S.part[(2 * kMB + r) * KR + j] + S.part[(3 * kMB + r) * KR + j]);
      }
      __syncthreads();
      if (tid == 0) {
        if (A.trace) A.trace[2 * (size_t)it + 1] = mtime();
        __threadfence();
        atomicAdd(&A.pdone[I.front], 1);
        atomicAdd(A.done, 1);
      }
      continue;
    }
    if (I.blk == kMWhole) {
      mbwd_whole<KR>(A, I, S, tid);
    } else {
      const double* g = A.pool + I.goff;
      const int64_t ld = I.ld;
      const int32_t* rw = A.rows + I.rows_off;
      const int nr = I.nr, blk = I.blk, np = I.np, nf = I.nf;
      const int r0 = I.r0, lo = r0 + nr;
      mload_dinv<true>(S.D, A.dinv + I.doff + (int64_t)kMB * kMB * blk, nr, tid);
      for (int idx = tid; idx < nr * KR; idx += kMT) S.w[idx] = A.y[(int64_t)(I.start + r0) * KR + idx];
      double acc[KR];
#pragma unroll
      for (int j = 0; j < KR; ++j) acc[j] = 0.0;
      // contribution columns: the ancestors' x (final: the front is ready);
      // wide fronts have them in partial items instead (I.pad chunks)
      for (int base = I.pad > 0 ? nf : np; base < nf; base += kMStage) {
        const int hi = min(nf, base + kMStage);
        for (int idx = tid; idx < (hi - base) * KR; idx += kMT) {
          const int c = base + idx / KR, j = idx % KR;
          S.stg[idx] = __ldcg(&A.xnew[(int64_t)rw[c] * KR + j]);
        }
        __syncthreads();
        mstream<KR>(g + r0 + row, ld, row < nr, S.stg - base * KR, base, hi, grp, acc);
        __syncthreads();
      }
      // later pivot blocks of this front, published last first, consumed by value
      consume_blocks<KR, false>(A, A.xnew + (int64_t)I.start * KR, g + r0 + row, ld, row < nr, lo, np, S.stg, tid,
                                grp, acc);
      put_part<KR>(S.part, grp, row, acc);
      if (I.pad > 0 && tid == 0) {  // the front's partial items (queued ahead of its blocks)
        unsigned long long t0 = 0;
        while (ld_acq(&A.pdone[I.front]) < A.npart[I.front]) {
          __nanosleep(32);
          if (mstalled(A, t0)) break;
        }
      }
      __syncthreads();
      sub_parts<KR>(S.w, S.part, nr, tid);
      if (I.pad > 0)  // chunk partials in chunk order (deterministic)
        for (int idx = tid; idx < nr * KR; idx += kMT) {
          double t = 0.0;
          for (int k = 0; k < I.pad; ++k) t += __ldcg(&A.bpart[(int64_t)I.cbvec_off + (int64_t)k * kMSlot + idx]);
          S.w[idx] -= t;
        }
      __syncthreads();
      double out[KR / 4];
      tile_mul<KR>(S.D, S.w, nr, row, jq, out);
      if (row < nr)
#pragma unroll
        for (int t = 0; t < KR / 4; ++t) store_xm<KR>(A, I.start + r0 + row, jq * (KR / 4) + t, out[t]);
    }
    __syncthreads();
    if (A.trace && tid == 0) A.trace[2 * (size_t)it + 1] = mtime();
    if (I.blk == 0 || I.blk == kMWhole) {  // the front is complete: its effective children are ready
      if (tid == 0) __threadfence();
      __syncthreads();
      for (int x = tid; x < I.nech; x += kMT) {
        const int f = A.ech[I.ech_off + x];
        if (atomicSub(&A.deps[f], 1) == 1) {
          __threadfence();
          if (A.warp_items && A.fcnt[f] == 1 && mwarp_ok<KR>(A.items[A.fbase[f]])) {
            mpush_any<KR>(A, f);
          } else if (x == 0) {  // the first effective child's first item runs here next
            mpush(A, f, 1);
            keep_s = A.fbase[f];
          } else {
            mpush(A, f);
          }
        }
      }
    }
    __syncthreads();
    if (tid == 0) atomicAdd(A.done, 1);
  }
}

}  // namespace

// ---------------------------------------------------------------------------
struct MSolvePlan {
  int nfr = 0, n_fwd = 0, n_bwd = 0;
  DeviceBuffer d_items_f, d_items_b, d_meta, d_ech, d_state0, d_state, d_stall;
  DeviceBuffer d_y, d_x, d_cb;  // interleaved, sized for 8 right-hand sides
  DeviceBuffer d_bpart;         // backward partial sums of wide fronts
  int64_t st_dep_f = 0, st_dep_b = 0, st_q_f = 0, st_q_b = 0, st_qctl = 0, st_pub = 0;
  int64_t st_bl_f = 0, st_bl_b = 0, st_pc = 0;  // batch lists, per-level counters
  int64_t mt_bb_f = 0, mt_bb_b = 0, mt_cf4 = 0, mt_cf8 = 0, mt_cb4 = 0, mt_cb8 = 0;
  int nlev = 1;
  int grid4 = 148, grid8 = 148;
};

void MSolvePlanDeleter::operator()(MSolvePlan* p) const { delete p; }

constexpr int kMaxRhs = 8;

static void msolve_prepare(FactorEngine& fe) {
  SetupTrace tr("msolve_prepare");
  const Symbolic& S = fe.sym;
  auto P = std::unique_ptr<MSolvePlan, MSolvePlanDeleter>(new MSolvePlan);
  const int nfr = static_cast<int>(S.fronts.size());
  P->nfr = nfr;
  std::vector<int32_t> npb(nfr), doff(nfr), fbase_f(nfr), fcnt_f(nfr), fbase_b(nfr, 0), fcnt_b(nfr, 0), ech_off(nfr);
  std::vector<std::vector<int32_t>> echl(nfr);
  int64_t dtot = 0;
  for (int f = 0; f < nfr; ++f) {
    const Front& F = S.fronts[f];
    npb[f] = (F.npiv + kMB - 1) / kMB;
    doff[f] = static_cast<int32_t>(dtot);  // same layout as rqb_solve_prepare's diagonal-tile inverses
    for (int b = 0; b < npb[f]; ++b) {
      const int64_t nr = std::min(F.npiv, (b + 1) * kMB) - b * kMB;
      dtot += nr * nr;
    }
    if (npb[f] > 0) {
      int a = F.parent;
      while (a >= 0 && S.fronts[a].npiv == 0) a = S.fronts[a].parent;
      if (a >= 0) echl[a].push_back(f);
    }
  }
  std::vector<int32_t> ech;
  for (int f = 0; f < nfr; ++f) {
    ech_off[f] = static_cast<int32_t>(ech.size());
    ech.insert(ech.end(), echl[f].begin(), echl[f].end());
  }
  std::vector<int> lvl_count;
  for (const Front& F : S.fronts) {
    if (F.level >= static_cast<int>(lvl_count.size())) lvl_count.resize(F.level + 1, 0);
    ++lvl_count[F.level];
  }
  const int whole_min = std::getenv("RQB_MWHOLE_MIN") ? std::atoi(std::getenv("RQB_MWHOLE_MIN")) : 128;
  auto item = [&](int f, int r0, int r1, int blk) {
    const Front& F = S.fronts[f];
    const FrontDev& D = fe.fronts_h[f];
    MItem it{};
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
    it.parent = F.parent;
    it.rows_off = static_cast<int32_t>(D.rows_off);
    it.cbvec_off = static_cast<int32_t>(D.cbvec_off);
    it.ech_off = ech_off[f];
    it.nech = static_cast<int32_t>(echl[f].size());
    it.doff = doff[f];
    return it;
  };
  std::vector<MItem> fwd, bwd;
  std::vector<char> whole(nfr);
  // warp items (mwarp_ok): whole items with one pivot block whose nf x KR
  // staging fits a warp's slice; bit 0: KR <= 8, bit 1: KR = 4; level << 8
  static const bool warp_items = !std::getenv("RQB_MWARP") || std::atoi(std::getenv("RQB_MWARP")) != 0;
  auto wflags = [&](int f) {
    const Front& F = S.fronts[f];
    if (!warp_items || npb[f] != 1) return 0;
    const int b = (F.nf <= mwarp_nf<8>() ? 1 : 0) | (F.nf <= mwarp_nf<4>() ? 2 : 0);
    return b ? (b | (F.level << 8)) : 0;
  };
  for (int f = 0; f < nfr; ++f) {
    const Front& F = S.fronts[f];
    whole[f] = npb[f] <= 2 && F.nf <= kMWholeNf && lvl_count[F.level] >= whole_min;
    fbase_f[f] = static_cast<int32_t>(fwd.size());
    if (whole[f]) {
      fwd.push_back(item(f, 0, F.nf, kMWhole));
      fwd.back().pad = wflags(f);
    } else {
      for (int b = 0; b < npb[f]; ++b) fwd.push_back(item(f, b * kMB, std::min(F.npiv, (b + 1) * kMB), b));
      for (int r = F.npiv; r < F.nf; r += kMB) fwd.push_back(item(f, r, std::min(F.nf, r + kMB), -1));
    }
    fcnt_f[f] = static_cast<int32_t>(fwd.size()) - fbase_f[f];
  }
  std::vector<int32_t> npart(nfr, 0);
  int64_t pslots = 0;
  for (int f = nfr - 1; f >= 0; --f) {
    const Front& F = S.fronts[f];
    fbase_b[f] = static_cast<int32_t>(bwd.size());
    if (npb[f] > 0) {
      const int ncb = F.nf - F.npiv;
      if (whole[f]) {
        bwd.push_back(item(f, 0, F.npiv, kMWhole));
        bwd.back().pad = wflags(f);
      } else if (ncb > kMCbChunk) {
        // wide front: per pivot block, one partial item per kMCbChunk
        // contribution columns (independent, ahead of the blocks in the queue),
        // the block items add the partials in chunk order
        const int nck = (ncb + kMCbChunk - 1) / kMCbChunk;
        for (int b = npb[f] - 1; b >= 0; --b)
          for (int k = 0; k < nck; ++k) {
            MItem it = item(f, b * kMB, std::min(F.npiv, (b + 1) * kMB), kMPart);
            it.ech_off = k * kMCbChunk;
            it.nech = std::min(ncb, (k + 1) * kMCbChunk);
            it.cbvec_off = static_cast<int32_t>(pslots + (static_cast<int64_t>(b) * nck + k) * kMSlot);
            bwd.push_back(it);
          }
        for (int b = npb[f] - 1; b >= 0; --b) {
          MItem it = item(f, b * kMB, std::min(F.npiv, (b + 1) * kMB), b);
          it.pad = nck;
          it.cbvec_off = static_cast<int32_t>(pslots + static_cast<int64_t>(b) * nck * kMSlot);
          bwd.push_back(it);
        }
        npart[f] = npb[f] * nck;
        pslots += static_cast<int64_t>(npb[f]) * nck * kMSlot;
        if (pslots > INT32_MAX) throw Error(errc::solver, "multi-RHS solve: partial-sum slots exceed int32");
      } else {
        for (int b = npb[f] - 1; b >= 0; --b) bwd.push_back(item(f, b * kMB, std::min(F.npiv, (b + 1) * kMB), b));
      }
    }
    fcnt_b[f] = static_cast<int32_t>(bwd.size()) - fbase_b[f];
  }
  std::vector<int32_t> dfwd(nfr, 0), dbwd(nfr, 0);
  for (int f = 0; f < nfr; ++f) {
    const Front& F = S.fronts[f];
    for (int32_t c : F.children) dfwd[f] += fcnt_f[c];
    int a = F.parent;
    while (a >= 0 && S.fronts[a].npiv == 0) a = S.fronts[a].parent;
    dbwd[f] = a >= 0 ? 1 : 0;
  }
  std::vector<int32_t> qf(std::max<size_t>(1, fwd.size()), -1), qb(std::max<size_t>(1, bwd.size()), -1);
  int nq_f = 0, nq_b = 0;
  // batch lists: forward = initial batches (ready leaves eligible for both
  // KR, grouped by 8 here) + per-level regions; backward = per-level regions
  int nlev = 1;
  for (const Front& F : S.fronts) nlev = std::max(nlev, F.level + 1);
  std::vector<int32_t> blf, bbase_f(nlev, 0), bbase_b(nlev, 0), cf4(nlev, 0), cf8(nlev, 0), cb4(nlev, 0), cb8(nlev, 0);
  auto wpad = [](const std::vector<MItem>& v, int i) { return v[i].blk == kMWhole ? v[i].pad : 0; };
  for (int f = 0; f < nfr; ++f) {
    if (dfwd[f] == 0) {
      for (int i = 0; i < fcnt_f[f]; ++i) {
        const int it = fbase_f[f] + i;
        if (fcnt_f[f] == 1 && (wpad(fwd, it) & 1)) {
          blf.push_back(it);
          if (blf.size() % 8 == 0) qf[nq_f++] = -2 - (8 * static_cast<int>(blf.size() - 8) + 7);
        } else {
          qf[nq_f++] = it;
        }
      }
    } else if (fcnt_f[f] == 1) {
      const int pd = wpad(fwd, fbase_f[f]);
      if (pd & 1) ++cf8[pd >> 8];
      if (pd & 2) ++cf4[pd >> 8];
    }
    if (dbwd[f] == 0) {
      for (int i = 0; i < fcnt_b[f]; ++i) qb[nq_b++] = fbase_b[f] + i;
    } else if (fcnt_b[f] == 1) {
      const int pd = wpad(bwd, fbase_b[f]);
      if (pd & 1) ++cb8[pd >> 8];
      if (pd & 2) ++cb4[pd >> 8];
    }
  }
  if (blf.size() % 8) {
    const int r = static_cast<int>(blf.size() % 8);
    qf[nq_f++] = -2 - (8 * static_cast<int>(blf.size() - r) + r - 1);
  }
  int nbf = static_cast<int>(blf.size()), nbb = 0;
  for (int L = 0; L < nlev; ++L) {
    bbase_f[L] = nbf;
    nbf += cf4[L];  // KR = 4 counts bound KR = 8 (bit 0 implies bit 1)
    bbase_b[L] = nbb;
    nbb += cb4[L];
  }
  blf.resize(std::max(1, nbf), -1);
  std::vector<int32_t> blb(std::max(1, nbb), -1);
  P->n_fwd = static_cast<int>(fwd.size());
  P->n_bwd = static_cast<int>(bwd.size());
  if (fwd.empty()) fwd.push_back(MItem{});
  if (bwd.empty()) bwd.push_back(MItem{});
  if (ech.empty()) ech.push_back(0);
  P->d_items_f.upload(fwd.data(), sizeof(MItem) * fwd.size(), fe.stream);
  P->d_items_b.upload(bwd.data(), sizeof(MItem) * bwd.size(), fe.stream);
  std::vector<int32_t> meta;
  meta.insert(meta.end(), fbase_f.begin(), fbase_f.end());
  meta.insert(meta.end(), fcnt_f.begin(), fcnt_f.end());
  meta.insert(meta.end(), fbase_b.begin(), fbase_b.end());
  meta.insert(meta.end(), fcnt_b.begin(), fcnt_b.end());
  meta.insert(meta.end(), npart.begin(), npart.end());
  P->nlev = nlev;
  P->mt_bb_f = static_cast<int64_t>(meta.size());
  meta.insert(meta.end(), bbase_f.begin(), bbase_f.end());
  P->mt_bb_b = static_cast<int64_t>(meta.size());
  meta.insert(meta.end(), bbase_b.begin(), bbase_b.end());
  P->mt_cf4 = static_cast<int64_t>(meta.size());
  meta.insert(meta.end(), cf4.begin(), cf4.end());
  P->mt_cf8 = static_cast<int64_t>(meta.size());
  meta.insert(meta.end(), cf8.begin(), cf8.end());
  P->mt_cb4 = static_cast<int64_t>(meta.size());
  meta.insert(meta.end(), cb4.begin(), cb4.end());
  P->mt_cb8 = static_cast<int64_t>(meta.size());
  meta.insert(meta.end(), cb8.begin(), cb8.end());
  P->d_meta.upload(meta.data(), sizeof(int32_t) * meta.size(), fe.stream);
  P->d_ech.upload(ech.data(), sizeof(int32_t) * ech.size(), fe.stream);
  std::vector<int32_t> st;
  P->st_dep_f = 0;
  st.insert(st.end(), dfwd.begin(), dfwd.end());
  P->st_dep_b = static_cast<int64_t>(st.size());
  st.insert(st.end(), dbwd.begin(), dbwd.end());
  P->st_q_f = static_cast<int64_t>(st.size());
  st.insert(st.end(), qf.begin(), qf.end());
  P->st_q_b = static_cast<int64_t>(st.size());
  st.insert(st.end(), qb.begin(), qb.end());
  P->st_qctl = static_cast<int64_t>(st.size());
  st.insert(st.end(), {0, nq_f, 0, nq_b, 0, 0});  // {head, tail} fwd, bwd; items done fwd, bwd
  P->st_pub = static_cast<int64_t>(st.size());
  st.resize(st.size() + 3 * static_cast<size_t>(nfr), 0);  // published blocks fwd, bwd; bwd partials done
  P->st_bl_f = static_cast<int64_t>(st.size());
  st.insert(st.end(), blf.begin(), blf.end());
  P->st_bl_b = static_cast<int64_t>(st.size());
  st.insert(st.end(), blb.begin(), blb.end());
  P->st_pc = static_cast<int64_t>(st.size());
  st.resize(st.size() + 2 * static_cast<size_t>(nlev), 0);  // batch-list counters fwd, bwd
  P->d_state0.upload(st.data(), sizeof(int32_t) * st.size(), fe.stream);
  P->d_state.alloc(P->d_state0.bytes);
  P->d_stall.alloc(sizeof(int));
  RQB_CUDA(cudaMemsetAsync(P->d_stall.p, 0, sizeof(int), fe.stream));
  P->d_y.alloc(sizeof(double) * kMaxRhs * std::max<int64_t>(1, fe.n));
  P->d_x.alloc(sizeof(double) * kMaxRhs * std::max<int64_t>(1, fe.n));
  P->d_cb.alloc(sizeof(double) * kMaxRhs * std::max<int64_t>(1, S.cbvec));
  P->d_bpart.alloc(sizeof(double) * std::max<int64_t>(1, pslots));
  int nsm = 148, occ = 1;
  RQB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, fe.device));
  smem_at_least(mfwd_sweep<4, 3>, msmem_bytes<4>());
  smem_at_least(mbwd_sweep<4, 3>, msmem_bytes<4>());
  smem_at_least(mfwd_sweep<8, 2>, msmem_bytes<8>());
  smem_at_least(mbwd_sweep<8, 2>, msmem_bytes<8>());
  RQB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mfwd_sweep<4, 3>, kMT, msmem_bytes<4>()));
  P->grid4 = nsm * std::max(1, occ);
  RQB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mfwd_sweep<8, 2>, kMT, msmem_bytes<8>()));
  P->grid8 = nsm * std::max(1, occ);
  fe.mplan.reset(P.release());
  tr.mark("plan + uploads");
}

template <int KR, int kMinB>
static void msolve_launch(FactorEngine& fe, MArgs A, int grid) {
  MSolvePlan& P = *fe.mplan;
  cudaStream_t st = fe.stream;
  const int nfr = P.nfr;
  int* sb = P.d_state.as<int>();
  const int32_t* meta = P.d_meta.as<int32_t>();
  smem_at_least(mfwd_sweep<KR, kMinB>, msmem_bytes<KR>());
  smem_at_least(mbwd_sweep<KR, kMinB>, msmem_bytes<KR>());
  MArgs F = A;
  F.items = P.d_items_f.as<MItem>();
  F.nitems = P.n_fwd;
  F.deps = sb + P.st_dep_f;
  F.queue = sb + P.st_q_f;
  F.qctl = sb + P.st_qctl;
  F.done = sb + P.st_qctl + 4;
  F.pub = sb + P.st_pub;
  F.fbase = meta;
  F.fcnt = meta + nfr;
  F.blist = sb + P.st_bl_f;
  F.pcnt = sb + P.st_pc;
  F.bbase = meta + P.mt_bb_f;
  F.bcnt = meta + (KR == 4 ? P.mt_cf4 : P.mt_cf8);
  if (P.n_fwd > 0) mfwd_sweep<KR, kMinB><<<std::min(grid, P.n_fwd), kMT, msmem_bytes<KR>(), st>>>(F);
  MArgs B = A;
  if (A.trace) B.trace = A.trace + 2 * (size_t)P.n_fwd;
  B.items = P.d_items_b.as<MItem>();
  B.nitems = P.n_bwd;
  B.deps = sb + P.st_dep_b;
  B.queue = sb + P.st_q_b;
  B.qctl = sb + P.st_qctl + 2;
  B.done = sb + P.st_qctl + 5;
  B.pub = sb + P.st_pub + nfr;
  B.pdone = sb + P.st_pub + 2 * nfr;
  B.fbase = meta + 2 * nfr;
  B.fcnt = meta + 3 * nfr;
  B.npart = meta + 4 * nfr;
  B.blist = sb + P.st_bl_b;
  B.pcnt = sb + P.st_pc + P.nlev;
  B.bbase = meta + P.mt_bb_b;
  B.bcnt = meta + (KR == 4 ? P.mt_cb4 : P.mt_cb8);
  B.bpart = P.d_bpart.as<double>();
  if (P.n_bwd > 0) mbwd_sweep<KR, kMinB><<<std::min(grid, P.n_bwd), kMT, msmem_bytes<KR>(), st>>>(B);
  RQB_CUDA(cudaGetLastError());
}

void rqb_msolve_enqueue(FactorEngine& fe, const double* b, int64_t ldb, int nrhs, double* x, int64_t ldx,
                        double scale, const double* vu, int64_t ldv, double sigma, double* xl, int64_t b_row_stride) {
  if (nrhs <= 0) return;
  if (nrhs > kMaxRhs) fail(errc::config, "multi-RHS sweep: at most 8 right-hand sides per call");
  if (!fe.mplan) msolve_prepare(fe);
  MSolvePlan& P = *fe.mplan;
  cudaStream_t st = fe.stream;
  RQB_CUDA(cudaMemcpyAsync(P.d_state.p, P.d_state0.p, P.d_state0.bytes, cudaMemcpyDeviceToDevice, st));
  {  // published-by-value entries start unset (all-ones bit pattern)
    const size_t kr = nrhs <= 4 ? 4 : 8;
    RQB_CUDA(cudaMemsetAsync(P.d_y.p, 0xff, sizeof(double) * kr * fe.n, st));
    RQB_CUDA(cudaMemsetAsync(P.d_x.p, 0xff, sizeof(double) * kr * fe.n, st));
  }
  MArgs A{};
  A.ech = P.d_ech.as<int32_t>();
  A.gsrc = fe.d_gsrc.as<int4>();
  A.pool = fe.d_pool.as<double>();
  A.dinv = fe.d_dinv.as<double>();
  A.perm = fe.d_perm.as<int32_t>();
  A.rows = fe.d_rows.as<int32_t>();
  A.b = b;
  A.ldb = ldb;
  A.bsr = b_row_stride;
  A.y = P.d_y.as<double>();
  A.cbvec = P.d_cb.as<double>();
  A.xnew = P.d_x.as<double>();
  A.xout = x;
  A.ldx = ldx;
  A.scale = scale;
  A.vu = vu;
  A.ldv = ldv;
  A.sigma = sigma;
  A.xl = xl;
  A.nrhs = nrhs;
  A.warp_items = !std::getenv("RQB_MWARP") || std::atoi(std::getenv("RQB_MWARP")) != 0;
  A.stall = P.d_stall.as<int>();
  unsigned long long* trace = nullptr;
  {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (std::getenv("RQB_MSOLVE_TRACE") && cs == cudaStreamCaptureStatusNone)
      RQB_CUDA(cudaMalloc(&trace, sizeof(unsigned long long) * 2 * (size_t)(P.n_fwd + P.n_bwd)));
  }
  A.trace = trace;
  if (nrhs <= 4)
    msolve_launch<4, 3>(fe, A, P.grid4);
  else
    msolve_launch<8, 2>(fe, A, P.grid8);
  fe.launches_solve = 2;
  if (trace) {  // development trace: {n_fwd, n_bwd} then per item {start, end} (ns)
    cudaStreamSynchronize(st);
    std::vector<unsigned long long> h(2 * (size_t)(P.n_fwd + P.n_bwd));
    cudaMemcpy(h.data(), trace, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
    if (FILE* fp = std::fopen(std::getenv("RQB_MSOLVE_TRACE"), "wb")) {
      const int32_t hdr[2] = {P.n_fwd, P.n_bwd};
      std::fwrite(hdr, sizeof(hdr), 1, fp);
      std::fwrite(h.data(), sizeof(unsigned long long), h.size(), fp);
      std::fclose(fp);
    }
    cudaFree(trace);
  }
}

void rqb_msolve_prepare(FactorEngine& fe) {
  if (!fe.mplan) msolve_prepare(fe);
}

void rqb_msolve_check(FactorEngine& fe) {
  if (!fe.mplan) return;
  int stv = 0;
  RQB_CUDA(cudaMemcpyAsync(&stv, fe.mplan->d_stall.p, sizeof(int), cudaMemcpyDeviceToHost, fe.stream));
  RQB_CUDA(cudaStreamSynchronize(fe.stream));
  if (stv) {
    RQB_CUDA(cudaMemsetAsync(fe.mplan->d_stall.p, 0, sizeof(int), fe.stream));
    fail(errc::solver, "multi-RHS triangular sweep stalled (watchdog): a dependency of the solve never resolved");
  }
}

}  // namespace rqb
