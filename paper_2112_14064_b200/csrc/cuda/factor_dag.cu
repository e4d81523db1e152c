// SPDX-License-Identifier: Apache-2.0
// Numeric multifrontal LU of Q(sigma) as ONE persistent, dependency-driven
// kernel (lu_factorize; it replaces the per-pivot rank-1 loop
// of kern::elim_step, kernels.cpp:58-69).
//
// Task DAG (built on the host in a topological order: tree height, panel step,
// front; within a step the tiles the next panel needs come first = lookahead):
//   SMALL(f)           nf <= 160: children's extend-add + whole-front LU in
//                      shared memory (16-column panels factored by one warp with
//                      warp-shuffle threshold pivot search; DMMA trailing update)
//   ASM(f, b)          big front, 64-column block: children's extend-add (gather)
//   DIAG(f, s)         32x32 diagonal block of panel s, unpivoted (speculative),
//                      inv(L11) / inv(U11) to scratch, in-block multiplier check
//   ROWS(f, s, a)      64-row tile row below the block: L = A inv(U11); max|l|
//                      over fully-summed rows -> per-panel flag (panel backed up)
//   COLS(f, s, b)      64-column tile column right of the block: U12 = inv(L11) A12
//   UPD(f, s, a, b)    64x64 tile -= L21 U12 on FP64 tensor cores (mma.sync
//                      m16n8k4 f64 -> DMMA.8x8x4), for tiles that hold pivot
//                      rows or pivot columns (they feed later panels)
//   UPDCB(f, a, b)     64x64 tile of the contribution block (rows and columns
//                      past npiv): ONE update with K = npiv after the last
//                      panel (cp.async double-buffered K loop, DMMA), instead
//                      of one K = 32 read-modify-write per panel step
// The last of DIAG/ROWS/COLS of a panel to finish checks the flag. If every
// multiplier of a fully-summed row satisfies |l| <= 10 (1 - 1e-14), the
// threshold-0.1 rule would have kept every
// diagonal pivot, so the speculative panel IS the pivoted result. Otherwise
// that CTA waits for the pending trailing updates, restores the panel from its
// backup and redoes it with exact threshold partial pivoting (prefer the
// diagonal, ties -> lowest row, singular < 1e-300), full-row swaps and U12.
// Then it releases the panel to the UPD tasks.
// Dataflow scheduling: every task carries a count of unfinished predecessors
// (host-built template, copied in per factorization); a finishing task
// decrements its successors and the one that reaches zero is pushed on a global
// FIFO ready queue. CTAs pop queue slots in order and only ever run ready
// tasks: no task-level spinning, no level barriers, no per-panel launches
// (the persistent grid idles only when nothing is ready). Every slot is
// eventually filled (DAG), so the schedule cannot deadlock. Data produced
// inside the kernel is read with ld.global.cg (L1 bypass); publication is
// __threadfence + atomic.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>

#include <cub/cub.cuh>

#include "device.cuh"

namespace rqb {

namespace {

constexpr int kDT = 256;          // threads per CTA
constexpr int kPB = 16;           // small-front panel width
constexpr int kTile = 64;         // big-front tile edge
constexpr int kTSP = kTile + 4;   // padded smem stride of DMMA operand tiles
constexpr double kLmax = 10.0 * (1.0 - 1e-14);  // 1/threshold, conservative
constexpr int kAsmRowTiles = 8;  // parent rows per extend-add task: 8 tiles
// ROWS / COLS tasks cover up to kRCMax tiles (one row / column per thread:
// with 64-row tiles only a quarter of the CTA worked and every tile paid the
// task's fixed latency); DagArgs::rc_group <= kRCMax at run time
constexpr int kRCMax = 4;
constexpr int kCnt = 7;  // per-front counters: tasks, asm, diag, rc, released, batches running, fallback
constexpr int kCntRun = 5, kCntFb = 6;
// Two configurations of the persistent kernel, chosen per factorization
// (rqb_dag_build): small problems are critical-path bound and want big SMALL
// fronts (nf <= 160 factored whole in 206 KB of shared memory, one CTA per
// SM); large problems are throughput bound and want two CTAs per SM (task
// latency of one hidden behind the other: 113 KB of shared memory and 128
// registers each, SMALL fronts up to nf = 256 whose pivot cross fits 112 KB).
constexpr int kSmallNfLatency = 160;
// throughput variant: fronts up to nf = 208 whose pivot cross fits 112 KB. Measured
// (resident factor, ms; 208 / 256 = every front a CTA's 256 threads can take):
// cfg4_riga 24.8 / 25.5, cfg4_iga 54.9 / 59.3 (a 220..256-row front as ONE CTA's
// SMALL task holds up its parent for > 100 us; tiled, its tasks spread over the
// grid), cfg5_p2..p5_riga, cfg5_p4_iga, cfg3_riga within 0.5%
constexpr int kSmallNfThroughput = 208;
constexpr size_t kSmallBytesLatency = 160 * 161 * 8;     // 206 KB: one CTA per SM
constexpr size_t kSmallBytesThroughput = 118 * 119 * 8;  // 112 KB: two CTAs per SM
constexpr double kThroughputFlops = 2e9;  // F_LU above which the two-CTA variant is used

enum : int16_t { T_SMALL = 0, T_ASM = 1, T_DIAG = 2, T_ROWS = 3, T_COLS = 4, T_UPD = 5, T_UPDCB = 6, T_UPDB = 7 };

struct Task {
  int32_t front;
  int16_t type, step;
  int32_t a, b;
};

struct FrontDag {
  int32_t tiles;       // tiles per dimension (big fronts), 0 for small
  int32_t tile_off;    // offset into tile_step[]
  int32_t ntasks;      // completion target of cnt[0]
  int32_t nasm;
  int32_t rc_off;      // offset into rc_prefix[] (steps + 1 entries)
  int32_t flag_off;    // offset into flagbits[] (one per step)
  int32_t slot;        // scratch slot (inverses), -1 small
  int32_t bnd_off;     // per child: (tiles + 1) first child CB column of each 64-column block
  int32_t task_base;   // first task of this front
  int32_t sb_off;      // offset into step_base[] (steps + 1 entries)
  int32_t parent;      // parent front (-1 root)
  int32_t acb;         // first contribution-block tile (rows / columns >= npiv)
  int32_t cb_base;     // first UPDCB task ((tiles - acb)^2 of them, row-major)
  int32_t ub_off;      // offset into ubase[] (tiles^2): first UPDB task of each pivot-region tile
  int64_t backup_off;  // panel backup nf x 32, then A12 backup 32 x nf
};

struct DagArgs {
  const FrontDev* fronts;
  const FrontDag* dag;
  const Task* tasks;
  int ntasks;
  int nqueued;  // tasks that pass through the ready queue (DIAG of steps >= 1 never do)
  const int32_t* inv;
  const int32_t* rel;   // child CB row -> parent-local row (FrontDev::rel_off)
  const int32_t* bnd;   // FrontDag::bnd_off
  double* pool;
  int32_t* ipiv;
  double* scratch;
  double* backup;
  int* cnt;
  int* tile_step;
  const int32_t* rc_prefix;
  unsigned long long* flagbits;
  int* flags;   // [0] singular, [1] swaps, [2] stall watchdog (1 queue, 2 fallback wait)
  int small_nf; // SMALL threshold of this plan (stride of the per-CTA panel backup)
  unsigned long long* prof;  // optional: per task type {work cycles, wait cycles, count}
  unsigned long long* trace; // optional (RQB_DAG_TRACE): per task {start, end} globaltimer ns
  double* small_backup;      // per CTA: 160 x 16 panel backup of the SMALL path
  int* deps;                 // remaining predecessors per task
  int* queue;                // ready queue (task ids, -1 = not yet pushed)
  int* qctl;                 // {head, tail}
  const int32_t* step_base;  // FrontDag::sb_off: first task of every panel step
  int upd_cp16;              // UPD operands by 16-byte cp.async (RQB_UPD_CP16=0: 8-byte copies)
  int upd_batch;             // deferred updates: panel steps per UPDB task (0: every update per step)
  int upd_tma;               // UPDCB / UPDB operand stages by TMA bulk copies (RQB_UPD_TMA=1)
  int rc_group;              // tiles per ROWS / COLS task (1 .. kRCMax)
  int upd_la;                // lookahead: the last upd_la steps before a tile's panel stay per step
  const int32_t* ubase;      // FrontDag::ub_off
  // lazy assembly: the SMALL / ASM task that owns a pool region zeroes it and
  // writes the original entries that land there (no pool memset, no separate
  // scatter launch): entries ent_beg[t] .. ent_end[t] - 1 of task t
  int keep_small;            // a SMALL parent runs in the CTA that completed its last child
  int lazy;
  const double* aval;        // Q(sigma) values (CSR order)
  const int* arrived;        // chunks of the upload sequence present in aval (streamed upload; see scatter_entries)
  const int32_t* ent_need;   // per task: chunks that must have arrived
  const int32_t* init_list;  // fed initial tasks (see the feeder in factor_dag_kernel); nullptr: all queued at the start
  int ninit;
  const int32_t* ent_src;    // CSR entry of each sorted position
  const int64_t* ent_dst;    // its pool offset
  const int32_t* ent_beg;
  const int32_t* ent_end;
};

// Deferred updates of a pivot-region tile: its updates from steps
// 0 .. lim - 1 run as UPDB tasks of upd_batch steps each (K = 32 upd_batch,
// the UPDCB code over a K range); steps >= lim stay per step (UPD), so the
// lookahead tiles on the panel chain keep their K = 32 latency. Must match
// rqb_dag_build.
__device__ __forceinline__ int upd_lim(const DagArgs& A, int a, int b, int steps) {
  return A.upd_batch > 0 ? min(steps, max(0, 2 * min(a, b) - A.upd_la)) : 0;
}


__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Spin waits give up after kStallNs (a dependency that never resolves is a
// bug): the watchdog flag makes every CTA leave and the host reports a stall
// instead of hanging the device.
constexpr unsigned long long kStallNs = 4000000000ull;

__device__ __forceinline__ bool spin_ge(const int* p, int target, int* flags) {
  if (*((volatile const int*)p) >= target) return true;
  const unsigned long long t0 = gtimer();
  while (*((volatile const int*)p) < target) {
    __nanosleep(64);
    if (gtimer() - t0 > kStallNs || *((volatile int*)&flags[2])) {
      atomicCAS(&flags[2], 0, 2);
      return false;
    }
  }
  return true;
}

__device__ __forceinline__ bool spin_le(const int* p, int target, int* flags) {
  const unsigned long long t0 = gtimer();
  while (*((volatile const int*)p) > target) {
    __nanosleep(64);
    if (gtimer() - t0 > kStallNs || *((volatile int*)&flags[2])) {
      atomicCAS(&flags[2], 0, 2);
      return false;
    }
  }
  return true;
}

__device__ __forceinline__ void dmma(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ double block_max(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double m = 0.0;
  for (int i = 0; i < kDT / 32; ++i) m = fmax(m, red[i]);
  __syncthreads();
  return m;
}

// Children's Schur blocks into front F (child-centric scatter, atomic-free:
// rel is injective, children are applied one after the other). For child ch
// only its CB columns [lo[ch], hi[ch]) and CB rows [rlo[ch], rhi[ch]) are
// applied; parent column c lives at dst + c * ldd (shared or global memory). Latency: a warp takes four child
// columns x 128 rows per iteration, all 32 loads (16 child values, 16 parent
// values) in flight before the first add.
__device__ void extend_add(const DagArgs& A, const FrontDev& F, const int* lo, const int* hi,
                           const int* rlo, const int* rhi, double* dst, int64_t ldd, bool dst_global) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kW = kDT / 32, kC = 4, kU = 4;
  for (int ch = 0; ch < F.nchild; ++ch) {
    const FrontDev C = A.fronts[ch == 0 ? F.child0 : F.child1];
    const int32_t* rel = A.rel + C.rel_off;
    const int ncb = C.nf - C.npiv;
    const double* cp = A.pool + C.off + C.npiv + (int64_t)C.npiv * C.ld;  // CB block origin
    for (int ic0 = lo[ch] + warp * kC; ic0 < hi[ch]; ic0 += kW * kC) {
      const double* src[kC];
      double* dcol[kC];
#pragma unroll
      for (int j = 0; j < kC; ++j) {
        const int ic = min(ic0 + j, hi[ch] - 1);
        src[j] = cp + (int64_t)ic * C.ld;
        dcol[j] = dst + (int64_t)__ldg(&rel[ic]) * ldd;
      }
      const int ncol = min(kC, hi[ch] - ic0);
      for (int k0 = rlo[ch]; k0 < rhi[ch]; k0 += 32 * kU) {
        int pr[kU];
        double v[kC][kU], d[kC][kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int kk = k0 + lane + 32 * u;
          pr[u] = kk < rhi[ch] ? __ldg(&rel[kk]) : -1;
        }
#pragma unroll
        for (int j = 0; j < kC; ++j)
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const bool ok = j < ncol && pr[u] >= 0;
            v[j][u] = ok ? __ldcg(&src[j][k0 + lane + 32 * u]) : 0.0;
            d[j][u] = ok ? (dst_global ? __ldcg(&dcol[j][pr[u]]) : dcol[j][pr[u]]) : 0.0;
          }
#pragma unroll
        for (int j = 0; j < kC; ++j)
#pragma unroll
          for (int u = 0; u < kU; ++u)
            if (j < ncol && pr[u] >= 0) dcol[j][pr[u]] = d[j][u] + v[j][u];
      }
    }
    __syncthreads();  // two children may touch the same entries
  }
}

// asynchronous 8-byte global -> shared copy (L1-allocating: the front's
// region was written by the scatter kernel, never read before in this launch)
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}

// ---------------------------------------------------------------------------
// dst(r, c) -= sum_{k0 <= k < k0 + kw} L(r, k) U(k, c) over r in [r0, r1),
// c in [c0, c1), DMMA on 16 x 32 warp tiles: L(r, k) = Lb[r + k * ldl],
// U(k, c) = Ub[k + (c - uoff) * ldu], dst(r, c) = D[r + (c - doff) * ldd]
// (shared memory, or the front in global memory when kGlobal).
__device__ __forceinline__ void cp_async8z(double* smem, const double* gmem, bool valid) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = valid ? 8 : 0;  // src-size 0: zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "r"(n) : "memory");
}

// 16-byte cp.async of two consecutive doubles, `n` of them valid (zero fill)
__device__ __forceinline__ void cp_async16z(double* smem, const double* gmem, int n) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(8 * n) : "memory");
}
template <bool kGlobal>
__device__ __forceinline__ void cross_update(const double* Lb, int ldl, const double* Ub, int ldu, int uoff,
                                             double* D, int64_t ldd, int doff, int r0, int r1, int c0,
                                             int c1, int k0, int kw, bool rd = true) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int mt = (r1 - r0 + 15) / 16, nt = (c1 - c0 + 31) / 32;
  for (int tile = warp; tile < mt * nt; tile += kDT / 32) {
    const int rr = r0 + (tile % mt) * 16, cc = c0 + (tile / mt) * 32;
    double acc[4][4], cv[4][4];
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[y][e] = 0.0;
    if (kGlobal)  // destination values in flight during the K loop
#pragma unroll
      for (int y = 0; y < 4; ++y)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = rr + gid + (e >> 1) * 8, c = cc + y * 8 + 2 * tig + (e & 1);
          cv[y][e] = (rd && r < r1 && c < c1) ? __ldcg(&D[r + (int64_t)(c - doff) * ldd]) : 0.0;
        }
    const int ra = rr + gid, rb = rr + gid + 8;
#pragma unroll 4
    for (int kk = 0; kk < kw; kk += 4) {
      const int kc = k0 + kk + tig;
      const bool kin = kk + tig < kw;
      const double a0 = (kin && ra < r1) ? Lb[ra + kc * ldl] : 0.0;
      const double a1 = (kin && rb < r1) ? Lb[rb + kc * ldl] : 0.0;
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int cb = cc + y * 8 + gid;
        const double b0 = (kin && cb < c1) ? Ub[kc + (cb - uoff) * ldu] : 0.0;
        dmma(acc[y], a0, a1, b0);
      }
    }
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = rr + gid + (e >> 1) * 8, c = cc + y * 8 + 2 * tig + (e & 1);
        if (r < r1 && c < c1) {
          double* p = &D[r + (int64_t)(c - doff) * ldd];
          *p = (kGlobal ? cv[y][e] : *p) - acc[y][e];
        }
      }
  }
}

// Zero rows [r0, r1) x columns [c0, c1) of front F and write the original
// entries task t owns (lazy assembly, see DagArgs::lazy). Ends with a barrier.
__device__ void zero_region(const DagArgs& A, const FrontDev& F, int r0, int r1, int c0, int c1) {
  double* g = A.pool + F.off;
  const int64_t ld = F.ld;
  const int nr = r1 - r0, nc = c1 - c0;
  if (((r0 | nr) & 1) == 0) {  // column segments of even length from an even row: 16-byte stores
    const int hr = nr >> 1;
    for (int idx = threadIdx.x; idx < hr * nc; idx += kDT) {
      const int r = 2 * (idx % hr), c = idx / hr;
      *reinterpret_cast<double2*>(&g[(r0 + r) + (int64_t)(c0 + c) * ld]) = make_double2(0.0, 0.0);
    }
  } else {
    for (int idx = threadIdx.x; idx < nr * nc; idx += kDT) {
      const int r = idx % nr, c = idx / nr;
      g[(r0 + r) + (int64_t)(c0 + c) * ld] = 0.0;
    }
  }
}

// Original entries of task t. When the values stream in from the host while
// the kernel runs (FactorEngine::factor_streamed) thread 0 first waits until
// the chunks holding the task's entries have arrived: ent_need[t] chunks of
// the upload sequence, `arrived` counts the chunks uploaded so far
// (0x7f7f7f7f when the values are resident). The
// values are read through L2 (the copy engine writes there; a line may also
// hold a neighbour task's values that arrive later).
__device__ void scatter_entries(const DagArgs& A, int t) {
  const int e0 = A.ent_beg[t], e1 = A.ent_end[t];
  if (threadIdx.x == 0 && e1 > e0) {
    const int need = __ldg(&A.ent_need[t]);
    int got;
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(got) : "l"(A.arrived) : "memory");
    if (got < need) {
      const unsigned long long t0 = gtimer();
      for (;;) {
        __nanosleep(256);
        asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(got) : "l"(A.arrived) : "memory");
        if (got >= need) break;
        if (gtimer() - t0 > kStallNs || *((volatile int*)&A.flags[2])) {
          atomicCAS(&A.flags[2], 0, 2);
          break;
        }
      }
    }
  }
  __syncthreads();
  for (int i = e0 + threadIdx.x; i < e1; i += kDT) A.pool[__ldg(&A.ent_dst[i])] = __ldcg(&A.aval[__ldg(&A.ent_src[i])]);
  __syncthreads();
}

__device__ void assemble_region(const DagArgs& A, const FrontDev& F, int t, int r0, int r1, int c0, int c1) {
  zero_region(A, F, r0, r1, c0, c1);
  scatter_entries(A, t);
}

// SMALL front (nf <= 256 = one thread per row): the pivot "cross" lives in
// shared memory — the column block Cb (all nf rows x npiv columns) and the row
// block Rb (npiv rows x the ncb contribution columns) — so the shared memory
// need is npiv (2 nf - npiv) doubles instead of nf^2. Children's Schur blocks
// are added in global memory first, the cross is factored with 16-column
// panels (one warp-shuffle-free row per thread, speculative unpivoted panel
// with exact threshold-pivoted redo), and the contribution block gets ONE
// K = npiv DMMA update straight from the cross to global memory.
__device__ void small_front(const DagArgs& A, const FrontDev& F, double* sm, int* piv_sh) {
  const int nf = F.nf, np = F.npiv;
  const int ldc = nf | 1, ldr = np | 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* g = A.pool + F.off;
  const int64_t ld = F.ld;
  // development profile (RQB_DAG_TRACE-free): sub-phase SM cycles in prof[24..29]
  long long tph = A.prof ? clock64() : 0;
  auto phase = [&](int k) {
    if (A.prof && threadIdx.x == 0) {
      const long long t = clock64();
      atomicAdd(&A.prof[24 + k], (unsigned long long)(t - tph));
      tph = t;
    }
  };
  double* Cb = sm;                             // (r, c < np)   -> Cb[r + c * ldc]
  double* Rb = sm + (int64_t)ldc * np;         // (r < np, c >= np) -> Rb[r + (c - np) * ldr]
  if (F.nchild > 0) {
    int lo[2] = {0, 0}, hi[2] = {0, 0};
    hi[0] = A.fronts[F.child0].nf - A.fronts[F.child0].npiv;
    if (F.nchild > 1) hi[1] = A.fronts[F.child1].nf - A.fronts[F.child1].npiv;
    extend_add(A, F, lo, hi, lo, hi, g, ld, true);  // ends with a barrier
  }
  phase(1);
  // the cross in flight at once (one latency); the lines were never read
  // through L1 in this launch (extend_add reads with ld.cg)
  for (int c = warp; c < nf; c += kDT / 32) {
    const int rows = c < np ? nf : np;
    double* dst = c < np ? Cb + (int64_t)c * ldc : Rb + (int64_t)(c - np) * ldr;
    for (int r = lane; r < rows; r += 32) cp_async8(&dst[r], &g[r + (int64_t)c * ld]);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  phase(2);
  __shared__ double red_s[kDT / 32];
  __shared__ double urow_s[2][kPB];
  __shared__ int any_swap_s;
  double* pbk = A.small_backup + (int64_t)blockIdx.x * A.small_nf * kPB;
  auto at = [&](int r, int c) -> double& { return c < np ? Cb[r + c * ldc] : Rb[r + (c - np) * ldr]; };
  for (int k0 = 0; k0 < np; k0 += kPB) {
    const int pw = min(kPB, np - k0);
    // ---- speculative unpivoted panel: thread t owns row t in registers; the
    //      pivot row is published in a double-buffered shared row (1 barrier/column)
    double lm = 0.0;
    bool sing = false;
    {
      const int i = tid;
      const bool own = i >= k0 && i < nf;
      double a[kPB];
#pragma unroll
      for (int c = 0; c < kPB; ++c) a[c] = (own && c < pw) ? Cb[i + (k0 + c) * ldc] : 0.0;
      if (own)
#pragma unroll
        for (int c = 0; c < kPB; ++c)
          if (c < pw) pbk[i + c * A.small_nf] = a[c];
#pragma unroll
      for (int jj = 0; jj < kPB; ++jj) {
        if (jj < pw) {
          double* ub = urow_s[jj & 1];
          if (i == k0 + jj)
#pragma unroll
            for (int c = 0; c < kPB; ++c) ub[c] = a[c];
          __syncthreads();
          const double ujj = ub[jj];
          sing = sing || !(fabs(ujj) >= kSingularTiny);
          if (own && i > k0 + jj) {
            const double l = a[jj] * (1.0 / ujj);
            a[jj] = l;
            if (i < np) lm = fmax(lm, fabs(l));
#pragma unroll
            for (int c = jj + 1; c < kPB; ++c) a[c] -= l * ub[c];
          }
        }
      }
      if (own)
#pragma unroll
        for (int c = 0; c < kPB; ++c)
          if (c < pw) Cb[i + (k0 + c) * ldc] = a[c];
    }
    __syncthreads();
    if (sing) lm = 1e300;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lm = fmax(lm, __shfl_xor_sync(0xffffffffu, lm, o));
    if (lane == 0) red_s[warp] = lm;
    if (tid == 0) any_swap_s = 0;
    __syncthreads();
    double lmax = 0.0;
    for (int q = 0; q < kDT / 32; ++q) lmax = fmax(lmax, red_s[q]);
    if (lmax <= kLmax) {
      if (tid < pw) {
        A.ipiv[F.start + k0 + tid] = k0 + tid;
        piv_sh[tid] = k0 + tid;
      }
    } else {
      // restore the panel, redo it with exact threshold pivoting (warp 0)
      if (tid < nf && tid >= k0)
        for (int c = 0; c < pw; ++c) Cb[tid + (k0 + c) * ldc] = pbk[tid + c * A.small_nf];
      __syncthreads();
      if (tid == 0) any_swap_s = 1;
    }
    __syncthreads();
    if (any_swap_s && warp == 0) {
      for (int j = k0; j < k0 + pw; ++j) {
        double best = -1.0;
        int bi = j;
        for (int i = j + lane; i < np; i += 32) {
          const double v = fabs(Cb[i + j * ldc]);
          if (v > best) best = v, bi = i;
        }
        warp_argmax(best, bi);
        const double diag = fabs(Cb[j + j * ldc]);
        int p = diag >= kPivThreshold * best ? j : bi;
        if (!(best >= kSingularTiny)) {
          if (lane == 0) atomicOr(&A.flags[0], 1);
          p = j;
        }
        if (lane == 0) {
          A.ipiv[F.start + j] = p;
          piv_sh[j - k0] = p;
          if (p != j) atomicAdd(&A.flags[1], 1);
        }
        if (p != j && lane < pw) {
          const int c = k0 + lane;
          const double t = Cb[j + c * ldc];
          Cb[j + c * ldc] = Cb[p + c * ldc];
          Cb[p + c * ldc] = t;
        }
        __syncwarp();
        const double ujj = Cb[j + j * ldc];
        for (int i = j + 1 + lane; i < nf; i += 32) {
          const double l = Cb[i + j * ldc] / ujj;
          Cb[i + j * ldc] = l;
          for (int c = j + 1; c < k0 + pw; ++c) Cb[i + c * ldc] -= l * Cb[j + c * ldc];
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (any_swap_s)  // pivot rows (< np) swapped across the other columns of the cross
      for (int c = tid; c < nf; c += kDT) {
        if (c >= k0 && c < k0 + pw) continue;
        for (int jj = 0; jj < pw; ++jj) {
          const int p = piv_sh[jj], j = k0 + jj;
          if (p != j) {
            const double t = at(j, c);
            at(j, c) = at(p, c);
            at(p, c) = t;
          }
        }
      }
    __syncthreads();
    // U12 = inv(L11) A12 over the panel rows, all columns right of the panel
    for (int c = k0 + pw + tid; c < nf; c += kDT) {
      double u[kPB];
#pragma unroll
      for (int jj = 0; jj < kPB; ++jj) u[jj] = jj < pw ? at(k0 + jj, c) : 0.0;
#pragma unroll
      for (int jj = 1; jj < kPB; ++jj) {
        double sv = u[jj];
#pragma unroll
        for (int t = 0; t < jj; ++t) sv -= Cb[k0 + jj + (k0 + t) * ldc] * u[t];
        u[jj] = sv;
      }
#pragma unroll
      for (int jj = 0; jj < kPB; ++jj)
        if (jj < pw) at(k0 + jj, c) = u[jj];
    }
    __syncthreads();
    // trailing update of the cross only: pivot columns (all rows) and the
    // pivot rows of the contribution columns
    const int t0 = k0 + pw;
    if (t0 < np) cross_update<false>(Cb, ldc, Cb, ldc, 0, Cb, ldc, 0, t0, nf, t0, np, k0, pw);
    if (t0 < np && np < nf) cross_update<false>(Cb, ldc, Rb, ldr, np, Rb, ldr, np, t0, np, np, nf, k0, pw);
    __syncthreads();
  }
  phase(3);
  for (int c = warp; c < nf; c += kDT / 32) {
    const int rows = c < np ? nf : np;
    const double* src = c < np ? Cb + (int64_t)c * ldc : Rb + (int64_t)(c - np) * ldr;
    for (int r = lane; r < rows; r += 32) g[r + (int64_t)c * ld] = src[r];
  }
  phase(4);
  // contribution block: one K = npiv pass, operands from the cross
  // (a leaf's contribution block holds no original entries and was not
  // zeroed, DagArgs::lazy == 2: written as -L21 U12 without the read)
  if (np < nf) cross_update<true>(Cb, ldc, Rb, ldr, np, g, ld, 0, np, nf, np, nf, 0, np, !(A.lazy == 2 && F.nchild == 0));
  if (A.prof) __syncthreads();
  phase(5);
}

// DIAG: 32x32 diagonal block of panel s, unpivoted (speculative), in the
// registers of warp 0 (row `lane` per thread; shuffles broadcast the pivot row).
// The factored block goes back to the front; ROWS/COLS solve against it.
// Code size matters here: every task type lives in one persistent kernel, so
// the panel tasks below are written as rolled loops (a fully unrolled 32-step
// substitution is tens of KB of SASS and thrashes the instruction cache).

// DIAG: unpivoted LU of the w x w diagonal block in shared memory, all
// threads: thread (i = tid & 31, columns cb + 8q) updates its 4 entries of row
// i per step (one barrier per step); the multipliers of column j are scaled
// after the barrier (the next step does not read column j).
__device__ void diag_task(const DagArgs& A, const FrontDev& F, const FrontDag& D, int s, double* sm) {
  const int k = s * kNB, w = min(kNB, F.npiv - k);
  double* g = A.pool + F.off;
  const int64_t ld = F.ld;
  const int tid = threadIdx.x, i = tid & 31, cb = tid >> 5;
  double* T = sm;  // 32 x 33
  double* red = sm + 32 * 33;
  double* bk = A.backup + D.backup_off;
  {
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = cb + 8 * q;
      v[q] = (i < w && c < w) ? __ldcg(&g[(k + i) + (int64_t)(k + c) * ld]) : (i == c ? 1.0 : 0.0);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = cb + 8 * q;
      T[i + c * 33] = v[q];
      if (i < w && c < w) bk[(k + i) + (int64_t)c * F.nf] = v[q];
    }
  }
  __syncthreads();
  double lm = 0.0;
  bool sing = false;
#pragma unroll 1
  for (int j = 0; j < w; ++j) {
    const double ujj = T[j + j * 33];
    if (!(fabs(ujj) >= kSingularTiny)) sing = true;
    const double rinv = 1.0 / ujj;
    if (i > j && i < w) {
      const double l = T[i + j * 33] * rinv;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = cb + 8 * q;
        if (c > j && c < w) T[i + c * 33] = fma(-l, T[j + c * 33], T[i + c * 33]);
      }
    }
    __syncthreads();
    if (tid < w && tid > j) {
      const double l = T[tid + j * 33] * rinv;
      T[tid + j * 33] = l;
      lm = fmax(lm, fabs(l));
    }
  }
  if (sing) lm = 1e300;  // forces the exact pivoted fallback (singular detection there)
  __syncthreads();
  lm = block_max(lm, red);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = cb + 8 * q;
    if (i < w && c < w) g[(k + i) + (int64_t)(k + c) * ld] = T[i + c * 33];
  }
  for (int j = tid; j < w; j += kDT) A.ipiv[F.start + k + j] = k + j;
  if (tid == 0) atomicMax(&A.flagbits[D.flag_off + s], (unsigned long long)__double_as_longlong(lm));
}

// ROWS: rows of tile row a below the diagonal block: solve L21 U11 = A21 row by
// row (forward substitution with the factored block), track max|l| over the
// fully-summed rows (threshold verification), back the panel rows up first.
__device__ void rows_task(const DagArgs& A, const FrontDev& F, const FrontDag& D, int s, int a,
                          double* sm, int ntl) {
  const int k = s * kNB, w = min(kNB, F.npiv - k), np = F.npiv;
  const int r0 = max(a * kTile, k + w), r1 = min((a + ntl) * kTile, F.nf);
  const int nr = r1 - r0;  // <= kRCMax * 64 = kDT: one row per thread
  double* g = A.pool + F.off;
  const int64_t ld = F.ld;
  const int tid = threadIdx.x;
  constexpr int kPS = kRCMax * kTile + 1;  // stride of the panel rows block
  double* P = sm;                 // up to 256 rows x 32 columns
  double* U = sm + kPS * kNB;     // 32 x 33 factored diagonal block
  double* red = U + 32 * 33;
  double* bk = A.backup + D.backup_off;
  {
    double vu[4], vp[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + i * kDT, r = idx % 32, c = idx / 32;
      vu[i] = (r < w && c < w) ? __ldcg(&g[(k + r) + (int64_t)(k + c) * ld]) : (r == c ? 1.0 : 0.0);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + i * kDT;
      U[(idx % 32) + (idx / 32) * 33] = vu[i];
    }
    // the panel rows, kTile x 32 per round (a round's loads all in flight;
    // measured: one cp.async pass over all rounds was slower)
    for (int t = 0; t < ntl; ++t) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int idx = tid + i * kDT, r = t * kTile + idx % kTile, c = idx / kTile;
        vp[i] = (r < nr && c < w) ? __ldcg(&g[(r0 + r) + (int64_t)(k + c) * ld]) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int idx = tid + i * kDT, r = t * kTile + idx % kTile, c = idx / kTile;
        P[r + c * kPS] = vp[i];
        if (r < nr && c < w) bk[(r0 + r) + (int64_t)c * F.nf] = vp[i];
      }
    }
  }
  __syncthreads();
  double lm = 0.0;
  if (tid < nr) {
    // x U11 = p, right-looking: x_j = s_j * (1/u_jj), then s_c -= x_j u_jc
    // (serial chain: one multiply + one FMA per column; the reciprocals are
    // independent of it)
    double x[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = P[tid + j * kPS];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      x[j] = j < w ? x[j] * (1.0 / U[j + j * 33]) : 0.0;
#pragma unroll
      for (int c = j + 1; c < 32; ++c) x[c] = fma(-x[j], U[j + c * 33], x[c]);
    }
    const bool cand = r0 + tid < np;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < w) {
        g[(r0 + tid) + (int64_t)(k + j) * ld] = x[j];
        if (cand) lm = fmax(lm, fabs(x[j]));
      }
  }
  lm = block_max(lm, red);
  if (tid == 0) atomicMax(&A.flagbits[D.flag_off + s], (unsigned long long)__double_as_longlong(lm));
}

// COLS: columns of tile column b right of the block: U12 = inv(L11) A12 by
// forward substitution with the unit-lower factored block (column per thread).
__device__ void cols_task(const DagArgs& A, const FrontDev& F, const FrontDag& D, int s, int b,
                          double* sm, int ntl) {
  const int k = s * kNB, w = min(kNB, F.npiv - k);
  const int c0 = max(b * kTile, k + w), c1 = min((b + ntl) * kTile, F.nf);
  const int nc = c1 - c0;
  double* g = A.pool + F.off;
  const int64_t ld = F.ld;
  const int tid = threadIdx.x;
  double* P = sm;               // 32 rows x up to 256 columns (P[r + c*33])
  double* L = sm + kRCMax * kTile * 33;  // 32 x 33 factored diagonal block
  double* bk2 = A.backup + D.backup_off + (int64_t)F.nf * kNB;
  {
    double vl[4], vp[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + i * kDT, r = idx % 32, c = idx / 32;
      vl[i] = (r < w && c < w) ? __ldcg(&g[(k + r) + (int64_t)(k + c) * ld]) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + i * kDT;
      L[(idx % 32) + (idx / 32) * 33] = vl[i];
    }
    for (int t = 0; t < ntl; ++t) {  // 32 x kTile per round
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int idx = tid + i * kDT, r = idx % kNB, c = t * kTile + idx / kNB;
        vp[i] = (r < w && c < nc) ? __ldcg(&g[(k + r) + (int64_t)(c0 + c) * ld]) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int idx = tid + i * kDT, r = idx % kNB, c = t * kTile + idx / kNB;
        P[r + c * 33] = vp[i];
        if (r < w && c < nc) bk2[r + (int64_t)(c0 + c) * kNB] = vp[i];
      }
    }
  }
  __syncthreads();
  if (tid < nc) {
    // L11 x = p (unit lower), right-looking: x_i final, then s_r -= l_ri x_i
    double x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = P[i + tid * 33];
#pragma unroll
    for (int i = 0; i < 32; ++i)
#pragma unroll
      for (int r = i + 1; r < 32; ++r) x[r] = fma(-L[r + i * 33], x[i], x[r]);
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < w) g[(k + i) + (int64_t)(c0 + tid) * ld] = x[i];
  }
}

constexpr int kBLD = kNB + 4;  // UPD / UPDCB: B stage stored [n][kk] (conflict-free fragment reads)

__device__ void upd_task(const DagArgs& A, const FrontDev& F, int s, int a, int b, double* sm) {
  const int k = s * kNB, w = min(kNB, F.npiv - k);
  const int r0 = max(a * kTile, k + w), r1 = min(a * kTile + kTile, F.nf);
  const int c0 = max(b * kTile, k + w), c1 = min(b * kTile + kTile, F.nf);
  double* g = A.pool + F.off;
  const int64_t ld = F.ld;
  double* As = sm;              // [kk][m]
  double* Bs = sm + kNB * kTSP; // [n][kk], stride kBLD
  const int tid = threadIdx.x;
  const int nr = r1 - r0, nc = c1 - c0;
  const int lane = tid & 31, warp = tid >> 5;  // 8 warps: 2 (m) x 4 (n) of 32 x 16
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  const int gid = lane >> 2, tig = lane & 3;
  // every global load of the task in flight at once: the A and B panels by
  // 16-byte cp.async straight into shared memory (B stored [n][kk]), this
  // thread's C fragment into registers
  double cv[2][2][4];
  if ((r0 & 1) == 0 && A.upd_cp16) {  // 16-byte source alignment (r0 = k + w can be odd after the last panel)
#pragma unroll
    for (int i = 0; i < kNB * kTile / 2 / kDT; ++i) {
      const int idx = tid + i * kDT;
      const int kk = idx / (kTile / 2), m = 2 * (idx % (kTile / 2));
      const int n = kk < w ? max(0, min(2, nr - m)) : 0;
      cp_async16z(&As[kk * kTSP + m], n ? &g[(r0 + m) + (int64_t)(k + kk) * ld] : g, n);
    }
  } else {
#pragma unroll
    for (int i = 0; i < kNB * kTile / kDT; ++i) {
      const int idx = tid + i * kDT;
      const int kk = idx / kTile, m = idx % kTile;
      const bool ok = kk < w && m < nr;
      cp_async8z(&As[kk * kTSP + m], ok ? &g[(r0 + m) + (int64_t)(k + kk) * ld] : g, ok);
    }
  }
#pragma unroll
  for (int i = 0; i < kNB * kTile / 2 / kDT; ++i) {
    const int idx = tid + i * kDT;
    const int kk = 2 * (idx % (kNB / 2)), c = idx / (kNB / 2);
    const int n = c < nc ? max(0, min(2, w - kk)) : 0;
    cp_async16z(&Bs[c * kBLD + kk], n ? &g[(k + kk) + (int64_t)(c0 + c) * ld] : g, n);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = wm + x * 16 + gid + (e >> 1) * 8, c = wn + y * 8 + 2 * tig + (e & 1);
        cv[x][y][e] = (r < nr && c < nc) ? __ldcg(&g[(r0 + r) + (int64_t)(c0 + c) * ld]) : 0.0;
      }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  double acc[2][2][4];
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[x][y][e] = 0.0;
  const int ksteps = (w + 3) / 4;
  for (int ks = 0; ks < ksteps; ++ks) {
    const int kr = ks * 4 + tig;
    double af[2][2], bf[2];
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      af[x][0] = As[kr * kTSP + wm + x * 16 + gid];
      af[x][1] = As[kr * kTSP + wm + x * 16 + gid + 8];
    }
#pragma unroll
    for (int y = 0; y < 2; ++y) bf[y] = Bs[(wn + y * 8 + gid) * kBLD + kr];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) dmma(acc[x][y], af[x][0], af[x][1], bf[y]);
  }
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = wm + x * 16 + gid + (e >> 1) * 8, c = wn + y * 8 + 2 * tig + (e & 1);
        if (r < nr && c < nc) g[(r0 + r) + (int64_t)(c0 + c) * ld] = cv[x][y][e] - acc[x][y][e];
      }
}



// TMA bulk copies (cp.async.bulk, the copy engine: UBLKCP) completing on a
// shared-memory mbarrier (transaction bytes)
__device__ __forceinline__ void mbar_init(unsigned long long* mb, int count) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(mb));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* mb, unsigned bytes) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(mb));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mb, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(mb));
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}\n" ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, unsigned long long* mb) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const unsigned m = static_cast<unsigned>(__cvta_generic_to_shared(mb));
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
               "l"(gmem), "r"(bytes), "r"(m) : "memory");
}

// Contribution-block tile (a, b): C -= L(rows a, 0:npiv) U(0:npiv, cols b) in
// one pass, K in chunks of 32 staged by cp.async (two buffers: the next chunk
// is in flight while DMMA consumes the current one), C read once and written
// once. Runs after the front's last panel is released: every L and U column
// is final (pivot swaps never touch contribution-block rows).
__device__ void updcb_task(const DagArgs& A, const FrontDev& F, int a, int b, double* sm, int kb = 0,
                           int ke = -1) {
  const int r0 = a * kTile, r1 = min(r0 + kTile, F.nf);
  const int c0 = b * kTile, c1 = min(c0 + kTile, F.nf);
  const int K = ke < 0 ? F.npiv : ke;  // pivots kb .. K - 1
  double* g = A.pool + F.off;
  const int64_t ld = F.ld;
  const int tid = threadIdx.x;
  const int nr = r1 - r0, nc = c1 - c0;
  const int lane = tid & 31, warp = tid >> 5;  // 8 warps: 2 (m) x 4 (n) of 32 x 16
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  const int gid = lane >> 2, tig = lane & 3;
  // stage: As [kk][m] (stride kTSP) then Bs [n][kk] (stride kBLD), filled by
  // 16-byte cp.async (pairs along m of an L column, along kk of a U column)
  // with zero fill; with RQB_UPD_TMA=1 full 64 x 64 tiles and full 32-pivot
  // chunks arrive by TMA bulk copies instead (warp 0 issues the 32 L column
  // segments of 512 B and the 64 U column segments of 256 B, completion on the
  // stage's mbarrier)
  constexpr int kStage = kNB * kTSP + kTile * kBLD;
  __shared__ unsigned long long mbar[2];
  // measured (cfg4_riga): 96 bulk transfers of 256 / 512 B per chunk are slower
  // than 256 threads of 16-byte cp.async (UPDCB tile 18.8 -> 29.4 us, factor
  // 25.5 -> 28.5 ms), so the bulk path is opt-in (RQB_UPD_TMA=1)
  const bool bulk_tile = A.upd_tma && nr == kTile && nc == kTile;
  auto bulk_chunk = [&](int chunk) { return bulk_tile && kb + (chunk + 1) * kNB <= K; };
  if (bulk_tile) {
    if (tid == 0) {
      mbar_init(&mbar[0], 1);
      mbar_init(&mbar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  auto issue = [&](int chunk, int buf) {
    double* As = sm + buf * kStage;
    double* Bs = As + kNB * kTSP;
    const int k0 = kb + chunk * kNB;
    if (bulk_chunk(chunk)) {
      if (tid < 32) {  // warp 0: one L column segment and two U column segments per lane
        if (tid == 0) mbar_expect_tx(&mbar[buf], kNB * kTile * 8 * 2);
        // the stage was last read through the generic proxy
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        bulk_g2s(&As[tid * kTSP], &g[r0 + (int64_t)(k0 + tid) * ld], kTile * 8, &mbar[buf]);
        bulk_g2s(&Bs[tid * kBLD], &g[k0 + (int64_t)(c0 + tid) * ld], kNB * 8, &mbar[buf]);
        bulk_g2s(&Bs[(tid + 32) * kBLD], &g[k0 + (int64_t)(c0 + tid + 32) * ld], kNB * 8, &mbar[buf]);
      }
      return;
    }
#pragma unroll
    for (int i = 0; i < kNB * kTile / 2 / kDT; ++i) {
      const int idx = tid + i * kDT;
      const int kk = idx / (kTile / 2), m = 2 * (idx % (kTile / 2));
      const int n = (k0 + kk < K) ? max(0, min(2, nr - m)) : 0;
      cp_async16z(&As[kk * kTSP + m], n ? &g[(r0 + m) + (int64_t)(k0 + kk) * ld] : g, n);
    }
#pragma unroll
    for (int i = 0; i < kNB * kTile / 2 / kDT; ++i) {
      const int idx = tid + i * kDT;
      const int kk = 2 * (idx % (kNB / 2)), c = idx / (kNB / 2);
      const int n = c < nc ? max(0, min(2, K - k0 - kk)) : 0;
      cp_async16z(&Bs[c * kBLD + kk], n ? &g[(k0 + kk) + (int64_t)(c0 + c) * ld] : g, n);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int nchunks = (K - kb + kNB - 1) / kNB;
  issue(0, 0);
  double cv[2][2][4];
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = wm + x * 16 + gid + (e >> 1) * 8, c = wn + y * 8 + 2 * tig + (e & 1);
        cv[x][y][e] = (r < nr && c < nc) ? __ldcg(&g[(r0 + r) + (int64_t)(c0 + c) * ld]) : 0.0;
      }
  double acc[2][2][4];
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[x][y][e] = 0.0;
  for (int ch = 0; ch < nchunks; ++ch) {
    if (ch + 1 < nchunks) issue(ch + 1, (ch + 1) & 1);
    if (bulk_chunk(ch)) {
      mbar_wait(&mbar[ch & 1], (ch >> 1) & 1);
    } else if (ch + 1 < nchunks && !bulk_chunk(ch + 1)) {
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double* As = sm + (ch & 1) * kStage;
    const double* Bs = As + kNB * kTSP;
#pragma unroll
    for (int ks = 0; ks < kNB / 4; ++ks) {
      const int kr = ks * 4 + tig;
      double af[2][2], bf[2];
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        af[x][0] = As[kr * kTSP + wm + x * 16 + gid];
        af[x][1] = As[kr * kTSP + wm + x * 16 + gid + 8];
      }
#pragma unroll
      for (int y = 0; y < 2; ++y) bf[y] = Bs[(wn + y * 8 + gid) * kBLD + kr];
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y) dmma(acc[x][y], af[x][0], af[x][1], bf[y]);
    }
    __syncthreads();  // buffer (ch & 1) is refilled by the issue of chunk ch + 2
  }
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = wm + x * 16 + gid + (e >> 1) * 8, c = wn + y * 8 + 2 * tig + (e & 1);
        if (r < nr && c < nc) g[(r0 + r) + (int64_t)(c0 + c) * ld] = cv[x][y][e] - acc[x][y][e];
      }
}

// Exact threshold-pivoted redo of panel s (rare path, one CTA).
__device__ void panel_fallback(const DagArgs& A, const FrontDev& F, const FrontDag& D, int s,
                               double* sm, int* cnt) {
  const int k = s * kNB, w = min(kNB, F.npiv - k), np = F.npiv, nf = F.nf;
  double* g = A.pool + F.off;
  const int64_t ld = F.ld;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* red = sm;
  int* redi = reinterpret_cast<int*>(sm + 32);
  __shared__ int piv_s;
  // all per-step trailing updates of earlier panels must be in place (rows are
  // swapped across all columns). Tiles with deferred (UPDB) updates may still
  // owe some: a row swap moves their pending L rows with their C rows, so the
  // later batch stays consistent; only a batch running right now must not
  // overlap the swaps (fallback flag + running count, Dekker-style with the
  // UPDB start in factor_dag_kernel)
  if (tid == 0) {
    atomicExch(&cnt[kCntFb], 1);
    __threadfence();
    spin_le(&cnt[kCntRun], 0, A.flags);
    const int a0 = k / kTile, steps = (np + kNB - 1) / kNB;
    for (int a = a0; a < D.tiles; ++a)
      for (int b = a0; b < D.tiles; ++b)
        if ((a < D.acb || b < D.acb) && upd_lim(A, a, b, steps) <= s)  // per-step tiles
          spin_ge(&A.tile_step[D.tile_off + a * D.tiles + b], s, A.flags);
    __threadfence();
  }
  __syncthreads();
  const double* bk = A.backup + D.backup_off;
  const double* bk2 = bk + (int64_t)nf * kNB;
  for (int idx = tid; idx < (nf - k) * w; idx += kDT) {
    const int r = k + idx % (nf - k), c = idx / (nf - k);
    g[r + (int64_t)(k + c) * ld] = __ldcg(&bk[r + (int64_t)c * nf]);
  }
  for (int idx = tid; idx < (nf - k - w) * w; idx += kDT) {
    const int r = idx % w, c = k + w + idx / w;
    g[(k + r) + (int64_t)c * ld] = __ldcg(&bk2[r + (int64_t)c * kNB]);
  }
  __syncthreads();
  for (int j = k; j < k + w; ++j) {
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int i = j + tid; i < np; i += kDT) {
      const double v = fabs(__ldcg(&g[i + (int64_t)j * ld]));
      if (v > best) best = v, bi = i;
    }
    warp_argmax(best, bi);
    if (lane == 0) red[warp] = best, redi[warp] = bi;
    __syncthreads();
    if (tid == 0) {
      for (int q = 1; q < kDT / 32; ++q)
        if (red[q] > best || (red[q] == best && redi[q] < bi)) best = red[q], bi = redi[q];
      const double diag = fabs(__ldcg(&g[j + (int64_t)j * ld]));
      int p = diag >= kPivThreshold * best ? j : bi;
      if (!(best >= kSingularTiny)) {
        atomicOr(&A.flags[0], 1);
        p = j;
      }
      if (p != j) atomicAdd(&A.flags[1], 1);
      A.ipiv[F.start + j] = p;
      piv_s = p;
    }
    __syncthreads();
    const int p = piv_s;
    if (p != j) {
      for (int c = tid; c < nf; c += kDT) {
        const double t = __ldcg(&g[j + (int64_t)c * ld]);
        g[j + (int64_t)c * ld] = __ldcg(&g[p + (int64_t)c * ld]);
        g[p + (int64_t)c * ld] = t;
      }
      __syncthreads();
      // Row p's tile (ap, b) may still owe deferred steps ts .. s-1 (pending
      // UPDB batches; quiesced above) while row j's tile (s / 2, b) is current:
      // after the swap, bring position j up to date and give position p back
      // the debt its tile's batches will pay (same L rows, swapped with C)
      const int ap = p / kTile;
      if (A.upd_batch > 0 && ap != j / kTile)
        for (int c = k + w + tid; c < nf; c += kDT) {
          const int b = c / kTile;
          const int ts = *((volatile const int*)&A.tile_step[D.tile_off + ap * D.tiles + b]);
          if (ts >= s) continue;
          double dj = 0.0, dp = 0.0;
          for (int q = ts * kNB; q < k; ++q) {
            const double u = __ldcg(&g[q + (int64_t)c * ld]);
            dj = fma(__ldcg(&g[j + (int64_t)q * ld]), u, dj);
            dp = fma(__ldcg(&g[p + (int64_t)q * ld]), u, dp);
          }
          g[j + (int64_t)c * ld] = __ldcg(&g[j + (int64_t)c * ld]) - dj;
          g[p + (int64_t)c * ld] = __ldcg(&g[p + (int64_t)c * ld]) + dp;
        }
    }
    __syncthreads();
    const double ujj = __ldcg(&g[j + (int64_t)j * ld]);
    for (int i = j + 1 + tid; i < nf; i += kDT) {
      const double l = __ldcg(&g[i + (int64_t)j * ld]) / ujj;
      g[i + (int64_t)j * ld] = l;
      for (int c = j + 1; c < k + w; ++c)
        g[i + (int64_t)c * ld] = __ldcg(&g[i + (int64_t)c * ld]) - l * __ldcg(&g[j + (int64_t)c * ld]);
    }
    __syncthreads();
  }
  // U12 = inv(L11) A12 (forward substitution per column)
  for (int c = k + w + tid; c < nf; c += kDT)
    for (int jj = 1; jj < w; ++jj) {
      double sv = __ldcg(&g[(k + jj) + (int64_t)c * ld]);
      for (int t = 0; t < jj; ++t)
        sv -= __ldcg(&g[(k + jj) + (int64_t)(k + t) * ld]) * __ldcg(&g[(k + t) + (int64_t)c * ld]);
      g[(k + jj) + (int64_t)c * ld] = sv;
    }
  __syncthreads();
}

// Task index helpers (tasks of a front are contiguous; see rqb_dag_build)
__device__ __forceinline__ int a0_of(const FrontDev& F, int s) {
  const int k = s * kNB, w = min(kNB, F.npiv - k);
  return (k + w) / kTile;
}

// trailing tile rows/cols of step s (0 when the panel ends the front: npiv ==
// nf), identical to the host's task layout in rqb_dag_build
__device__ __forceinline__ int nr_of(const FrontDev& F, const FrontDag& D, int s) {
  const int k = s * kNB, t0 = k + min(kNB, F.npiv - k);
  return t0 < F.nf ? D.tiles - t0 / kTile : 0;
}

__device__ __forceinline__ int idx_diag(const DagArgs& A, const FrontDag& D, int s) {
  return A.step_base[D.sb_off + s];
}
// ROWS / COLS groups of step s: ceil(nr / rc_group) each
__device__ __forceinline__ int ngr_of(const DagArgs& A, const FrontDev& F, const FrontDag& D, int s) {
  return (nr_of(F, D, s) + A.rc_group - 1) / A.rc_group;
}
__device__ __forceinline__ int idx_rows(const DagArgs& A, const FrontDag& D, const FrontDev& F, int s,
                                         int a) {
  return A.step_base[D.sb_off + s] + 1 + (a - a0_of(F, s)) / A.rc_group;
}
__device__ __forceinline__ int idx_cols(const DagArgs& A, const FrontDag& D, const FrontDev& F, int s,
                                         int b) {
  const int a0 = a0_of(F, s);
  return A.step_base[D.sb_off + s] + 1 + ngr_of(A, F, D, s) + (b - a0) / A.rc_group;
}
// UPD tasks of step s: the trailing tiles (a, b) with a < acb or b < acb, in
// the order: pivot-region tile rows in full, then contribution-block rows
// restricted to pivot-region columns (same layout as rqb_dag_build)
__device__ __forceinline__ bool eager_tile(const FrontDag& D, int a, int b) { return a < D.acb || b < D.acb; }
__device__ __forceinline__ int idx_upd(const DagArgs& A, const FrontDag& D, const FrontDev& F, int s, int a,
                                        int b) {
  const int a0 = a0_of(F, s), nr = nr_of(F, D, s);
  const int np = max(0, D.acb - a0), x = a - a0, y = b - a0;
  const int base = A.step_base[D.sb_off + s] + 1 + 2 * ngr_of(A, F, D, s);
  return x < np ? base + x * nr + y : base + np * nr + (x - np) * np + y;
}

// One predecessor of task t completed: the last one pushes t on the ready queue.
// Ready queue: FIFO; a CTA claims the next slot (atomicAdd) and waits until a
// finishing task pushes into it.
__device__ __forceinline__ void notify(const DagArgs& A, int t) {
  if (atomicSub(&A.deps[t], 1) == 1) {
    __threadfence();
    const int slot = atomicAdd(&A.qctl[1], 1);
    atomicExch(&A.queue[slot], t);
  }
}

// release of panel step s for the eager tile (ua, ub): its per-step update,
// or the batch that ends at step s
__device__ __forceinline__ void release_tile(const DagArgs& A, const FrontDag& D, const FrontDev& F, int s,
                                             int steps, int ua, int ub) {
  const int lim = upd_lim(A, ua, ub, steps);
  if (s >= lim) {
    notify(A, idx_upd(A, D, F, s, ua, ub));
  } else {
    const int j = s / A.upd_batch;
    if (s == min((j + 1) * A.upd_batch, lim) - 1) notify(A, A.ubase[D.ub_off + ua * D.tiles + ub] + j);
  }
}

constexpr int kNopTask = 0x7fffffff;
__device__ int pop_task(const DagArgs& A) {
  const int h = atomicAdd(&A.qctl[0], 1);
  if (h >= A.nqueued) return -1;
  volatile int* q = A.queue;
  int t;
  if ((t = q[h]) < 0) {
    const unsigned long long t0 = gtimer();
    while ((t = q[h]) < 0) {
      __nanosleep(32);
      if (*((volatile int*)&A.flags[2])) return -1;
      if (gtimer() - t0 > kStallNs) {
        atomicCAS(&A.flags[2], 0, 1);
        return -1;
      }
    }
  }
  __threadfence();
  return t;
}

template <int kMinBlocks>
__global__ void __launch_bounds__(kDT, kMinBlocks) factor_dag_kernel(DagArgs A) {
  extern __shared__ double sm[];
  __shared__ int task_s, last_s, done_s, next_s;
  __shared__ int piv_sh[kPB];
  const int tid = threadIdx.x;
  if (tid == 0) next_s = -1;
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      const long long t0 = A.prof ? clock64() : 0;
      // DIAG(s + 1) runs in the CTA that finished its only predecessor (the
      // update of the diagonal tile): no queue round trip on the panel chain
      const int t = next_s >= 0 ? next_s : pop_task(A);
      next_s = -1;
      task_s = t;
      if (A.prof && t >= 0) atomicAdd(&A.prof[20], (unsigned long long)(clock64() - t0));
    }
    __syncthreads();
    const int t = task_s;
    if (t < 0) return;
    if (t == kNopTask) continue;  // slot of a task its predecessor's CTA kept
    const Task T = A.tasks[t];
    const int f = T.front;
    const FrontDev F = A.fronts[f];
    const FrontDag D = A.dag[f];
    int* cnt = A.cnt + kCnt * f;
    // feeder: only the first kInitWindow initial tasks (the leaves' SMALL / ASM
    // tasks) start in the ready queue; every one popped pushes the next of the
    // list, so tasks released during the run never queue up behind thousands
    // of leaves (whose entries may not have arrived yet when the values stream in)
    if (tid == 0 && A.init_list && (T.type == T_SMALL || T.type == T_ASM) && F.nchild == 0) {
      const int i = atomicAdd(&A.qctl[2], 1);
      if (i < A.ninit) {
        const int slot = atomicAdd(&A.qctl[1], 1);
        atomicExch(&A.queue[slot], __ldg(&A.init_list[i]));
      }
    }
    const long long t_work = A.prof ? clock64() : 0;
    if (A.trace && tid == 0) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
      A.trace[2 * (size_t)t] = gt;
    }
    // ---- work (every predecessor has completed: no waits)
    switch (T.type) {
      case T_SMALL: {
        const long long ta = A.prof ? clock64() : 0;
        if (A.lazy == 2 && F.nchild == 0 && F.npiv < F.nf) {  // leaf: only the pivot cross is zeroed
          zero_region(A, F, 0, F.ld, 0, F.npiv);
          zero_region(A, F, 0, F.npiv, F.npiv, F.nf);
          scatter_entries(A, t);
        } else if (A.lazy) {
          assemble_region(A, F, t, 0, F.ld, 0, F.nf);
        }
        if (A.prof && tid == 0) atomicAdd(&A.prof[24], (unsigned long long)(clock64() - ta));
        small_front(A, F, sm, piv_sh);
      }
        break;
      case T_ASM: {  // parent column block b, parent row block a (kAsmRowTiles tiles)
        if (A.lazy)
          assemble_region(A, F, t, T.a * kAsmRowTiles * kTile, min(F.ld, (T.a + 1) * kAsmRowTiles * kTile),
                          T.b * kTile, min(F.nf, (T.b + 1) * kTile));
        int lo[2] = {0, 0}, hi[2] = {0, 0}, rlo[2] = {0, 0}, rhi[2] = {0, 0};
        for (int ch = 0; ch < F.nchild; ++ch) {
          const int32_t* bd = A.bnd + D.bnd_off + ch * (D.tiles + 1);
          lo[ch] = bd[T.b];
          hi[ch] = bd[T.b + 1];
          rlo[ch] = bd[min(T.a * kAsmRowTiles, D.tiles)];
          rhi[ch] = bd[min((T.a + 1) * kAsmRowTiles, D.tiles)];
        }
        extend_add(A, F, lo, hi, rlo, rhi, A.pool + F.off, F.ld, true);
        break;
      }
      case T_DIAG: diag_task(A, F, D, T.step, sm); break;
      case T_ROWS: rows_task(A, F, D, T.step, T.a, sm, min(A.rc_group, a0_of(F, T.step) + nr_of(F, D, T.step) - T.a)); break;
      case T_COLS: cols_task(A, F, D, T.step, T.b, sm, min(A.rc_group, a0_of(F, T.step) + nr_of(F, D, T.step) - T.b)); break;
      case T_UPD: upd_task(A, F, T.step, T.a, T.b, sm); break;
      case T_UPDCB: updcb_task(A, F, T.a, T.b, sm); break;
      case T_UPDB: {  // steps [j B, min((j + 1) B, lim)) of tile (a, b)
        if (tid == 0) {  // not while a panel fallback swaps rows of this front (see panel_fallback)
          for (;;) {
            atomicAdd(&cnt[kCntRun], 1);
            __threadfence();
            if (atomicAdd(&cnt[kCntFb], 0) == 0) break;
            atomicSub(&cnt[kCntRun], 1);
            while (*((volatile int*)&cnt[kCntFb]) != 0) __nanosleep(256);
          }
        }
        __syncthreads();
        const int steps = (F.npiv + kNB - 1) / kNB;
        const int lim = upd_lim(A, T.a, T.b, steps);
        const int s0 = T.step * A.upd_batch, s1 = min(s0 + A.upd_batch, lim);
        updcb_task(A, F, T.a, T.b, sm, s0 * kNB, min(s1 * kNB, F.npiv));
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          atomicSub(&cnt[kCntRun], 1);
        }
        break;
      }
    }
    __syncthreads();
    if (A.trace && tid == 0) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
      A.trace[2 * (size_t)A.ntasks + 2 * (size_t)t] = gt;  // work done
    }
    if (tid == 0) __threadfence();
    __syncthreads();
    if (A.trace && tid == 0) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
      A.trace[2 * (size_t)A.ntasks + 2 * (size_t)t + 1] = gt;  // fence done
    }
    // ---- successors
    const int steps = (F.npiv + kNB - 1) / kNB;
    // tasks that never redo data after this point count towards front
    // completion right away (overlaps the round trip with the notifications)
    const bool early_done =
        T.type == T_SMALL || T.type == T_ASM || T.type == T_UPD || T.type == T_UPDCB || T.type == T_UPDB;
    if (early_done && tid == 160) done_s = (atomicAdd(&cnt[0], 1) + 1 == D.ntasks);
    if (T.type == T_DIAG || T.type == T_ROWS || T.type == T_COLS) {
      if (T.type == T_DIAG) {
        const int a0 = a0_of(F, T.step), nr = nr_of(F, D, T.step);
        for (int x = a0 + tid * A.rc_group; x < a0 + nr; x += kDT * A.rc_group) {  // one per group
          notify(A, idx_rows(A, D, F, T.step, x));
          notify(A, idx_cols(A, D, F, T.step, x));
        }
      }
      if (tid == 0) last_s = (atomicAdd(&cnt[3], 1) + 1 == A.rc_prefix[D.rc_off + T.step + 1]);
      __syncthreads();
      if (last_s) {  // last of the panel: verify, fall back if needed, release the updates
        if (tid == 0) __threadfence();
        __syncthreads();
        const unsigned long long bits = atomicAdd(&A.flagbits[D.flag_off + T.step], 0ull);
        if (!(__longlong_as_double((long long)bits) <= kLmax)) {
          panel_fallback(A, F, D, T.step, sm, cnt);
          __syncthreads();
          if (tid == 0) {
            __threadfence();  // publish the redone panel before releasing the updates
            atomicExch(&cnt[kCntFb], 0);  // deferred batches of this front may run again
          }
          __syncthreads();
        }
        const int a0 = a0_of(F, T.step), nr = nr_of(F, D, T.step);
        // lookahead first: the next panel's tile row and column, then the bulk
        for (int x = tid; x < 2 * nr - 1; x += kDT) {
          const int ua = x < nr ? a0 : a0 + (x - nr + 1), ub = x < nr ? a0 + x : a0;
          if (eager_tile(D, ua, ub)) release_tile(A, D, F, T.step, steps, ua, ub);
        }
        __syncthreads();
        for (int x = tid; x < (nr > 1 ? (nr - 1) * (nr - 1) : 0); x += kDT) {
          const int ua = a0 + 1 + x / (nr - 1), ub = a0 + 1 + x % (nr - 1);
          if (eager_tile(D, ua, ub)) release_tile(A, D, F, T.step, steps, ua, ub);
        }
        if (T.step == steps - 1) {  // last panel: the contribution block in one pass per tile
          const int ncb = D.tiles - D.acb;
          for (int x = tid; x < ncb * ncb; x += kDT) notify(A, D.cb_base + x);
        }
      }
    } else if (T.type == T_UPD) {
      // one notification per warp: the atomic round trips overlap
      const int s1 = T.step + 1;
      if (tid == 64) atomicAdd(&A.tile_step[D.tile_off + T.a * D.tiles + T.b], 1);
      if (s1 < steps && (tid & 31) == 0 && tid < 4 * 32 + 1) {
        const int a1 = a0_of(F, s1), an = (s1 * kNB) / kTile;
        const bool trail = nr_of(F, D, s1) > 0;  // step s1 has trailing rows / columns
        switch (tid >> 5) {
          case 0:  // tid 0: the next panel's diagonal block runs here next
            if (T.a == an && T.b == an) next_s = idx_diag(A, D, s1);
            break;
          case 1:
            if (trail && T.b == an && T.a >= a1) notify(A, idx_rows(A, D, F, s1, T.a));
            break;
          case 2:
            if (trail && T.a == an && T.b >= a1) notify(A, idx_cols(A, D, F, s1, T.b));
            break;
          case 3:
            if (trail && T.a >= a1 && T.b >= a1) notify(A, idx_upd(A, D, F, s1, T.a, T.b));
            break;
        }
      }
    } else if (T.type == T_ASM) {
      if (tid == 0 && steps > 0) notify(A, idx_diag(A, D, 0));
    } else if (T.type == T_UPDB && tid == 0) {
      const int lim = upd_lim(A, T.a, T.b, steps);
      const int s0 = T.step * A.upd_batch, s1 = min(s0 + A.upd_batch, lim);
      atomicAdd(&A.tile_step[D.tile_off + T.a * D.tiles + T.b], s1 - s0);
      if (s1 < lim)
        notify(A, A.ubase[D.ub_off + T.a * D.tiles + T.b] + T.step + 1);
      else if (lim < steps)
        notify(A, idx_upd(A, D, F, lim, T.a, T.b));
    }
    // front completion releases the parent's SMALL / ASM tasks
    if (!early_done && tid == 0) done_s = (atomicAdd(&cnt[0], 1) + 1 == D.ntasks);
    __syncthreads();
    if (done_s && D.parent >= 0) {
      const FrontDag PD = A.dag[D.parent];
      if (PD.tiles == 0) {
        // depth-first: the CTA that completes a SMALL parent's last child runs
        // the parent next (one child's Schur block is still hot in L2, and
        // when the values stream in the parents do not queue up behind leaves
        // whose entries have not arrived). The parent's queue slot is filled
        // with a no-op so the queue accounting (nqueued) stays exact.
        if (tid == 0) {
          if (A.keep_small) {
            if (atomicSub(&A.deps[PD.task_base], 1) == 1) {
              __threadfence();
              const int slot = atomicAdd(&A.qctl[1], 1);
              atomicExch(&A.queue[slot], kNopTask);
              next_s = PD.task_base;
            }
          } else {
            notify(A, PD.task_base);
          }
        }
      } else {
        for (int x = tid; x < PD.nasm; x += kDT) notify(A, PD.task_base + x);
      }
    }
    if (A.trace && tid == 0) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
      A.trace[2 * (size_t)t + 1] = gt;
    }
    if (tid == 0 && A.prof) {
      const long long t_end = clock64();
      const int slot = (T.type == T_UPDCB || T.type == T_UPDB) ? 21 : 3 * T.type;  // K-batched: 21..23
      atomicAdd(&A.prof[slot + 0], (unsigned long long)(t_end - t_work));
      atomicAdd(&A.prof[slot + 2], 1ull);
    }
  }
}

int div_up(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// owning task (SMALL or ASM) of every original entry's pool destination
__global__ void ent_key_k(int64_t nnz, const int64_t* __restrict__ qdst, const int64_t* __restrict__ foff,
                          const int32_t* __restrict__ fidx, int nfr, const FrontDev* __restrict__ fronts,
                          const FrontDag* __restrict__ dag, int32_t* __restrict__ key, int32_t* __restrict__ val) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = qdst[e];
    int lo = 0, hi = nfr;  // last front with foff <= d
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (foff[mid] <= d) lo = mid;
      else hi = mid;
    }
    const int f = fidx[lo];
    const FrontDev& F = fronts[f];
    const FrontDag& D = dag[f];
    const int64_t loc = d - F.off;
    const int c = static_cast<int>(loc / F.ld), r = static_cast<int>(loc % F.ld);
    key[e] = D.tiles == 0 ? D.task_base : D.task_base + (r / (kAsmRowTiles * kTile)) * D.tiles + c / kTile;
    val[e] = static_cast<int32_t>(e);
  }
}

__global__ void ent_bounds_k(int64_t n, const int32_t* __restrict__ key, int32_t* __restrict__ beg,
                             int32_t* __restrict__ end) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t k = key[i];
    if (i == 0 || key[i - 1] != k) beg[k] = static_cast<int32_t>(i);
    if (i == n - 1 || key[i + 1] != k) end[k] = static_cast<int32_t>(i + 1);
  }
}

// Streamed upload plan (FactorEngine::factor_streamed). The CSR values go up
// in chunks of `chunk` values; chunk_first_k: per chunk, the earliest position
// in the initial ready queue among the tasks owning one of its entries (the
// host sends the chunks in that order); ent_need_k: per task, how many chunks
// of that sequence must have arrived before its entries can be read.
__global__ void chunk_first_k(int64_t n, const int32_t* __restrict__ key, const int32_t* __restrict__ src,
                              const int32_t* __restrict__ rank, int64_t chunk, int32_t* __restrict__ first) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = rank[key[i]];
    const int c = static_cast<int>(src[i] / chunk);
    if (r < first[c]) atomicMin(&first[c], r);
  }
}

__global__ void ent_need_k(int64_t n, const int32_t* __restrict__ key, const int32_t* __restrict__ src,
                           const int32_t* __restrict__ seq, int64_t chunk, int32_t* __restrict__ need) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int v = seq[src[i] / chunk] + 1;
    int* p = &need[key[i]];
    if (v > *p) atomicMax(p, v);
  }
}

__global__ void gather_i64_k(int64_t n, const int32_t* __restrict__ idx, const int64_t* __restrict__ src,
                             int64_t* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

}  // namespace

struct DagPlan {
  DeviceBuffer d_tasks, d_dag, d_cnt, d_tile, d_rc, d_flagbits, d_backup, d_prof, d_bnd,
      d_small_backup, d_deps0, d_deps, d_queue0, d_queue, d_qctl, d_qctl0, d_sb, d_trace;
  int ntasks = 0, nqueued = 0, nfronts = 0, ntile = 0, nflag = 0, grid = 148, nready = 0;
  int occ = 1, small_nf = 160;  // kernel variant (see kSmallNfLatency / kSmallNfThroughput)
  int upd_batch = 0, upd_la = 2;  // deferred pivot-region updates (upd_lim)
  int rc_group = 1;               // tiles per ROWS / COLS task
  DeviceBuffer d_ubase;
  int lazy = 0;                   // lazy assembly (DagArgs::lazy)
  DeviceBuffer d_ent_src, d_ent_dst, d_ent_beg, d_ent_end, d_ent_need, d_init;
  int ninit = 0;  // initial tasks fed during the run (0: all in the queue at the start)
  std::vector<FrontDag> dag_h;   // host copy of the per-front plan (tile counts, acb)
  size_t smem = 0;
  double flops_upd = 0;
};

void rqb_dag_build(FactorEngine& fe) {
  const Symbolic& S = fe.sym;
  const int nfr = static_cast<int>(S.fronts.size());
  auto P = std::make_unique<DagPlan>();
  std::vector<FrontDag> dag(nfr);
  std::vector<int32_t> rc_prefix, bnd, step_base, deps;
  std::vector<Task> tasks;
  int tile_off = 0, flag_off = 0, slot = 0;
  int64_t backup = 0;
  int max_small = 0, nfused = 0;
  P->occ = S.flops_lu >= kThroughputFlops ? 2 : 1;
  if (const char* e = std::getenv("RQB_DAG_OCC")) P->occ = std::atoi(e) == 2 ? 2 : 1;
  int small_max = P->occ == 2 ? kSmallNfThroughput : kSmallNfLatency;
  if (const char* e = std::getenv("RQB_SMALL_NF")) small_max = std::min(kDT, std::atoi(e));
  // shared memory of a SMALL front: the pivot cross (see small_front)
  auto small_bytes = [](const Front& F) {
    const size_t ldc = F.nf | 1, ldr = F.npiv | 1;
    return sizeof(double) * (ldc * F.npiv + ldr * (F.nf - F.npiv));
  };
  const size_t small_budget = P->occ == 2 ? kSmallBytesThroughput : kSmallBytesLatency;
  size_t max_small_bytes = 0;
  // deferred contribution blocks pay in the throughput regime (cfg4_riga
  // factor 44.1 -> 36.3 ms); the latency variant keeps per-step updates, which
  // overlap the panel chain (cfg2_riga 0.85 -> 0.83 ms)
  int cb_min_steps = P->occ == 2 ? 1 : (1 << 30);
  if (const char* e = std::getenv("RQB_CB_MIN_STEPS")) cb_min_steps = std::atoi(e);
  // deferred pivot-region updates (UPDB, see upd_lim): the throughput variant
  // batches upd_batch panel steps per tile update and keeps the last upd_la
  // steps before a tile's own panel per step
  // measured (ms, group 1 / 2 / 4): cfg4_riga 26.3 / 25.3 / 25.3, cfg4_iga
  // 62.9 / 59.6 / 58.9, cfg5_p5_riga 11.8 / 11.0 / 10.9, cfg3_iga 4.94 / 4.93 /
  // 5.16 (its panel chain binds), cfg2_riga (latency variant) 0.83 / 0.84
  P->rc_group = P->occ == 2 ? (S.flops_lu >= 4e10 ? kRCMax : 2) : 1;
  if (const char* e = std::getenv("RQB_RC_GROUP")) P->rc_group = std::max(1, std::min(kRCMax, std::atoi(e)));
  // measured: cfg4_riga 28.3 -> 26.8 ms, cfg4_iga 68.6 -> 61.0 ms (4: 27.0 / 62.2); later, with the
  // current task set, 8 / 16 / 24: cfg4_riga 25.24 / 25.15 / 25.17, cfg4_iga 59.0 / 58.2 / 58.1 — kept
  // at 8: with 16 the changed factor rounding left the single-vector cfg3_iga nev = 50 solve stagnating
  // in its degenerate cluster
  P->upd_batch = P->occ == 2 ? 8 : 0;
  P->upd_la = 2;
  if (const char* e = std::getenv("RQB_UPD_BATCH")) P->upd_batch = std::max(0, std::atoi(e));
  if (const char* e = std::getenv("RQB_UPD_LOOKAHEAD")) P->upd_la = std::max(1, std::atoi(e));
  std::vector<int32_t> ubase;
  int ndead = 0;
  auto lim_of = [&](int a, int b, int steps) {
    return P->upd_batch > 0 ? std::min(steps, std::max(0, 2 * std::min(a, b) - P->upd_la)) : 0;
  };
  // tasks of a front are contiguous; fronts in postorder
  for (int f = 0; f < nfr; ++f) {
    const Front& F = S.fronts[f];
    FrontDag& D = dag[f];
    D.task_base = static_cast<int32_t>(tasks.size());
    D.slot = -1;
    D.parent = F.parent;
    const int nch = static_cast<int>(F.children.size());
    if (F.nf <= small_max && small_bytes(F) <= small_budget) {
      tasks.push_back({f, T_SMALL, 0, 0, 0});
      deps.push_back(nch);
      D.ntasks = 1;
      max_small = std::max(max_small, F.nf);
      max_small_bytes = std::max(max_small_bytes, small_bytes(F));
      continue;
    }
    D.tiles = div_up(F.nf, kTile);
    // contribution block deferred to one K = npiv pass per tile when the front
    // has at least cb_min_steps panels (else its tiles are updated per step)
    D.acb = div_up(F.npiv, kTile) < D.tiles && div_up(F.npiv, kNB) >= cb_min_steps ? div_up(F.npiv, kTile)
                                                                                      : D.tiles;
    D.tile_off = tile_off;
    tile_off += D.tiles * D.tiles;
    const int steps = div_up(F.npiv, kNB);
    D.flag_off = flag_off;
    flag_off += std::max(1, steps);
    D.slot = slot++;
    D.backup_off = backup;
    backup += 2LL * F.nf * kNB;
    D.nasm = D.tiles * div_up(D.tiles, kAsmRowTiles);
    int front_dead = 0;
    D.bnd_off = static_cast<int32_t>(bnd.size());
    for (int32_t c : F.children) {
      const Front& C = S.fronts[c];
      const int32_t* rel = fe.rel_h.data() + fe.fronts_h[c].rel_off;
      const int ncb = C.nf - C.npiv;
      for (int b = 0; b <= D.tiles; ++b)
        bnd.push_back(static_cast<int32_t>(std::lower_bound(rel, rel + ncb, b * kTile) - rel));
    }
    // extend-add tasks: 64-column block x kAsmRowTiles-tile row block of the
    // parent (children's rows are a sorted map: each parent block is a
    // contiguous child range, so concurrent tasks never touch the same entry)
    for (int a = 0; a < div_up(D.tiles, kAsmRowTiles); ++a)
      for (int b = 0; b < D.tiles; ++b) {
        tasks.push_back({f, T_ASM, 0, a, b});
        deps.push_back(nch);
      }
    D.rc_off = static_cast<int32_t>(rc_prefix.size());
    D.sb_off = static_cast<int32_t>(step_base.size());
    rc_prefix.push_back(0);
    int acc = 0;
    for (int s = 0; s < steps; ++s) {
      const int k = s * kNB, w = std::min(kNB, F.npiv - k), t0 = k + w;
      const int a0 = t0 / kTile;
      const int nr = t0 < F.nf ? D.tiles - a0 : 0;
      const int an = k / kTile;
      step_base.push_back(static_cast<int32_t>(tasks.size()));
      tasks.push_back({f, T_DIAG, (int16_t)s, an, an});
      deps.push_back(s == 0 ? D.nasm : 1);  // s >= 1: run by its predecessor's CTA, never queued
      if (s > 0) ++nfused;
      // ROWS / COLS groups of rc_group tiles: DIAG(s) + each tile's UPD(s - 1)
      const int G = P->rc_group, ngr = (nr + G - 1) / G;
      for (int a = a0; a < a0 + nr; a += G) {
        tasks.push_back({f, T_ROWS, (int16_t)s, a, an});
        deps.push_back(s == 0 ? 1 : 1 + std::min(G, a0 + nr - a));
      }
      for (int b = a0; b < a0 + nr; b += G) {
        tasks.push_back({f, T_COLS, (int16_t)s, an, b});
        deps.push_back(s == 0 ? 1 : 1 + std::min(G, a0 + nr - b));
      }
      // eager tiles (pivot rows or pivot columns), layout of idx_upd
      const int np = std::max(0, D.acb - a0);
      auto push_upd = [&](int a, int b) {
        tasks.push_back({f, T_UPD, (int16_t)s, a, b});
        if (s < lim_of(a, b, steps)) {  // this step's update runs inside an UPDB batch
          deps.push_back(1 << 30);
          ++ndead, ++front_dead;
          return;
        }
        deps.push_back(s == 0 ? 1 : 2);
        const double rr = std::min(F.nf, (a + 1) * kTile) - std::max(a * kTile, t0);
        const double cc = std::min(F.nf, (b + 1) * kTile) - std::max(b * kTile, t0);
        P->flops_upd += 2.0 * w * rr * cc;
      };
      for (int x = 0; x < std::min(np, nr); ++x)
        for (int y = 0; y < nr; ++y) push_upd(a0 + x, a0 + y);
      for (int x = np; x < nr; ++x)
        for (int y = 0; y < np; ++y) push_upd(a0 + x, a0 + y);
      acc += 1 + 2 * ngr;
      rc_prefix.push_back(acc);
    }
    step_base.push_back(static_cast<int32_t>(tasks.size()));
    // contribution-block tiles: one K = npiv update each, released by the last panel
    D.cb_base = static_cast<int32_t>(tasks.size());
    if (steps > 0)
      for (int a = D.acb; a < D.tiles; ++a)
        for (int b = D.acb; b < D.tiles; ++b) {
          tasks.push_back({f, T_UPDCB, 0, a, b});
          deps.push_back(1);
          const double rr = std::min(F.nf, (a + 1) * kTile) - a * kTile;
          const double cc = std::min(F.nf, (b + 1) * kTile) - b * kTile;
          P->flops_upd += 2.0 * F.npiv * rr * cc;
        }
    // deferred updates: per pivot-region tile, batches of upd_batch steps over
    // steps 0 .. lim - 1 (first batch released by its last panel, later ones
    // also by the previous batch of the tile)
    D.ub_off = static_cast<int32_t>(ubase.size());
    ubase.resize(ubase.size() + static_cast<size_t>(D.tiles) * D.tiles, -1);
    if (P->upd_batch > 0)
      for (int a = 0; a < D.tiles; ++a)
        for (int b = 0; b < D.tiles; ++b) {
          if (!(a < D.acb || b < D.acb)) continue;
          const int lim = lim_of(a, b, steps);
          if (lim <= 0) continue;
          ubase[D.ub_off + a * D.tiles + b] = static_cast<int32_t>(tasks.size());
          for (int j = 0; j * P->upd_batch < lim; ++j) {
            tasks.push_back({f, T_UPDB, (int16_t)j, a, b});
            deps.push_back(j == 0 ? 1 : 2);
            const int k0 = j * P->upd_batch * kNB, k1 = std::min(std::min((j + 1) * P->upd_batch, lim) * kNB, F.npiv);
            const double rr = std::min(F.nf, (a + 1) * kTile) - a * kTile;
            const double cc = std::min(F.nf, (b + 1) * kTile) - b * kTile;
            P->flops_upd += 2.0 * (k1 - k0) * rr * cc;
          }
        }
    D.ntasks = static_cast<int32_t>(tasks.size()) - D.task_base - front_dead;
  }
  // initial ready queue: tasks without predecessors (SMALL / ASM of leaf fronts)
  std::vector<int32_t> queue0(tasks.size(), -1);
  int nready = 0;
  for (size_t t = 0; t < tasks.size(); ++t)
    if (deps[t] == 0) queue0[nready++] = static_cast<int32_t>(t);
  P->nready = nready;
  P->ntasks = static_cast<int>(tasks.size());
  P->nqueued = P->ntasks - nfused - ndead;
  P->nfronts = nfr;
  P->ntile = std::max(1, tile_off);
  P->nflag = std::max(1, flag_off);
  if (rc_prefix.empty()) rc_prefix.push_back(0);
  if (step_base.empty()) step_base.push_back(0);
  if (bnd.empty()) bnd.push_back(0);
  if (tasks.empty()) {
    tasks.push_back({0, T_SMALL, 0, 0, 0});
    deps.push_back(0);
    queue0.assign(1, -1);
  }
  P->d_tasks.upload(tasks.data(), sizeof(Task) * tasks.size(), fe.stream);
  P->d_dag.upload(dag.data(), sizeof(FrontDag) * nfr, fe.stream);
  P->d_rc.upload(rc_prefix.data(), sizeof(int32_t) * rc_prefix.size(), fe.stream);
  P->d_bnd.upload(bnd.data(), sizeof(int32_t) * bnd.size(), fe.stream);
  P->d_sb.upload(step_base.data(), sizeof(int32_t) * step_base.size(), fe.stream);
  if (ubase.empty()) ubase.push_back(-1);
  P->d_ubase.upload(ubase.data(), sizeof(int32_t) * ubase.size(), fe.stream);
  P->d_deps0.upload(deps.data(), sizeof(int32_t) * deps.size(), fe.stream);
  P->d_deps.alloc(sizeof(int32_t) * deps.size());
  P->d_queue0.upload(queue0.data(), sizeof(int32_t) * queue0.size(), fe.stream);
  P->d_queue.alloc(sizeof(int32_t) * queue0.size());
  P->d_qctl.alloc(sizeof(int) * 4);
  {
    const int q0[4] = {0, nready, 0, 0};
    P->d_qctl0.upload(q0, sizeof(q0), fe.stream);
  }
  P->d_cnt.alloc(sizeof(int) * kCnt * nfr);
  P->d_tile.alloc(sizeof(int) * P->ntile);
  P->d_flagbits.alloc(sizeof(unsigned long long) * P->nflag);
  P->d_backup.alloc(sizeof(double) * std::max<int64_t>(1, backup));
  fe.d_scratch.alloc(sizeof(double) * std::max(1, slot) * 2 * kNB * kNB);
  const size_t small_smem = max_small_bytes;
  P->small_nf = std::max(1, max_small);
  const size_t tile_smem = sizeof(double) * std::max(4 * kNB * kTSP, 2 * (kNB * kTSP + kTile * kBLD));  // UPD / UPDCB: two stages
  const size_t rows_smem = sizeof(double) * std::max<size_t>((kRCMax * kTile + 1) * kNB + 33 * 32 + 64,
                                                             kRCMax * kTile * 33 + 33 * 32);
  const size_t diag_smem = sizeof(double) * (3 * 32 * 33 + 128);
  P->smem = std::max({small_smem, tile_smem, rows_smem, diag_smem, size_t(16 * 1024)});
  auto kern = P->occ == 2 ? factor_dag_kernel<2> : factor_dag_kernel<1>;
  smem_at_least(kern, P->smem);
  int nsm = 148, occ = 1;
  RQB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, fe.device));
  RQB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kDT, P->smem));
  P->grid = std::max(1, std::min(P->ntasks, nsm * std::max(1, occ)));
  P->d_small_backup.alloc(sizeof(double) * P->grid * P->small_nf * kPB);
  fe.dag_ntasks = P->ntasks;
  // lazy assembly: original entries grouped by the task that owns their destination
  // measured: cfg4_riga 26.8 -> 25.5 ms, cfg4_iga 61.3 -> 60.0 ms; the latency
  // variant keeps the pool memset + scatter (cfg2_riga 0.78 vs 0.81 ms lazy:
  // the zeroing sits on its critical path)
  P->lazy = P->occ == 2 ? 2 : 0;  // 2: leaf SMALL fronts zero only their pivot cross (1: whole fronts)
  if (const char* e = std::getenv("RQB_LAZY_ZERO")) P->lazy = std::atoi(e);
  if (P->lazy && fe.nnz > 0) {
    const int64_t nnz = fe.nnz;
    std::vector<std::pair<int64_t, int32_t>> fo(nfr);
    for (int q = 0; q < nfr; ++q) fo[q] = {fe.fronts_h[q].off, q};
    std::sort(fo.begin(), fo.end());
    std::vector<int64_t> foff(nfr);
    std::vector<int32_t> fidx(nfr);
    for (int q = 0; q < nfr; ++q) foff[q] = fo[q].first, fidx[q] = fo[q].second;
    DeviceBuffer d_foff, d_fidx, k0, k1, v0;
    d_foff.upload(foff.data(), sizeof(int64_t) * nfr, fe.stream);
    d_fidx.upload(fidx.data(), sizeof(int32_t) * nfr, fe.stream);
    k0.alloc(sizeof(int32_t) * nnz);
    k1.alloc(sizeof(int32_t) * nnz);
    v0.alloc(sizeof(int32_t) * nnz);
    P->d_ent_src.alloc(sizeof(int32_t) * nnz);
    P->d_ent_dst.alloc(sizeof(int64_t) * nnz);
    P->d_ent_beg.alloc(sizeof(int32_t) * P->ntasks);
    P->d_ent_end.alloc(sizeof(int32_t) * P->ntasks);
    RQB_CUDA(cudaMemsetAsync(P->d_ent_beg.p, 0, P->d_ent_beg.bytes, fe.stream));
    RQB_CUDA(cudaMemsetAsync(P->d_ent_end.p, 0, P->d_ent_end.bytes, fe.stream));
    const int blocks = static_cast<int>(std::min<int64_t>((nnz + 255) / 256, 148 * 32));
    ent_key_k<<<blocks, 256, 0, fe.stream>>>(nnz, fe.d_qdst.as<int64_t>(), d_foff.as<int64_t>(),
                                              d_fidx.as<int32_t>(), nfr, fe.d_fronts.as<FrontDev>(),
                                              P->d_dag.as<FrontDag>(), k0.as<int32_t>(), v0.as<int32_t>());
    RQB_CUDA(cudaGetLastError());
    int bits = 1;
    while ((1LL << bits) < P->ntasks) ++bits;
    size_t tmp_bytes = 0;
    RQB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0.as<int32_t>(), k1.as<int32_t>(),
                                             v0.as<int32_t>(), P->d_ent_src.as<int32_t>(), nnz, 0, bits,
                                             fe.stream));
    DeviceBuffer tmp;
    tmp.alloc(std::max<size_t>(tmp_bytes, 16));
    RQB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, k0.as<int32_t>(), k1.as<int32_t>(),
                                             v0.as<int32_t>(), P->d_ent_src.as<int32_t>(), nnz, 0, bits,
                                             fe.stream));
    ent_bounds_k<<<blocks, 256, 0, fe.stream>>>(nnz, k1.as<int32_t>(), P->d_ent_beg.as<int32_t>(),
                                                 P->d_ent_end.as<int32_t>());
    gather_i64_k<<<blocks, 256, 0, fe.stream>>>(nnz, P->d_ent_src.as<int32_t>(), fe.d_qdst.as<int64_t>(),
                                                 P->d_ent_dst.as<int64_t>());
    RQB_CUDA(cudaGetLastError());
    // ---- streamed upload plan: chunk sequence, per-task needs, and the
    // initial ready tasks (the leaves' SMALL / ASM tasks) in the order their
    // entries arrive, so a CTA waiting for its task's entries never holds
    // back a task whose entries are already there
    {
      if (const char* e = std::getenv("RQB_STREAM_CHUNK")) fe.stream_chunk = std::max<int64_t>(1 << 16, std::atoll(e));
      const int64_t chunk = fe.stream_chunk;
      const int nch = static_cast<int>((nnz + chunk - 1) / chunk);
      std::vector<int32_t> q(P->nready), rank(P->ntasks, 0x7fffffff);
      RQB_CUDA(cudaMemcpyAsync(q.data(), P->d_queue0.p, sizeof(int32_t) * P->nready, cudaMemcpyDeviceToHost, fe.stream));
      RQB_CUDA(cudaStreamSynchronize(fe.stream));
      for (int i = 0; i < P->nready; ++i) rank[q[i]] = i;
      DeviceBuffer d_rank, d_first, d_seq;
      d_rank.upload(rank.data(), sizeof(int32_t) * rank.size(), fe.stream);
      d_first.alloc(sizeof(int32_t) * nch);
      RQB_CUDA(cudaMemsetAsync(d_first.p, 0x7f, sizeof(int32_t) * nch, fe.stream));
      chunk_first_k<<<blocks, 256, 0, fe.stream>>>(nnz, k1.as<int32_t>(), P->d_ent_src.as<int32_t>(),
                                                    d_rank.as<int32_t>(), chunk, d_first.as<int32_t>());
      RQB_CUDA(cudaGetLastError());
      std::vector<int32_t> first(nch), seq(nch);
      RQB_CUDA(cudaMemcpyAsync(first.data(), d_first.p, sizeof(int32_t) * nch, cudaMemcpyDeviceToHost, fe.stream));
      RQB_CUDA(cudaStreamSynchronize(fe.stream));
      fe.chunk_order.resize(nch);
      std::iota(fe.chunk_order.begin(), fe.chunk_order.end(), 0);
      static const bool csr_order = std::getenv("RQB_STREAM_ORDER") && std::atoi(std::getenv("RQB_STREAM_ORDER")) == 0;
      if (!csr_order)
        std::stable_sort(fe.chunk_order.begin(), fe.chunk_order.end(),
                         [&](int32_t a, int32_t b) { return first[a] < first[b]; });
      for (int i = 0; i < nch; ++i) seq[fe.chunk_order[i]] = i;
      d_seq.upload(seq.data(), sizeof(int32_t) * nch, fe.stream);
      P->d_ent_need.alloc(sizeof(int32_t) * P->ntasks);
      RQB_CUDA(cudaMemsetAsync(P->d_ent_need.p, 0, sizeof(int32_t) * P->ntasks, fe.stream));
      ent_need_k<<<blocks, 256, 0, fe.stream>>>(nnz, k1.as<int32_t>(), P->d_ent_src.as<int32_t>(),
                                                 d_seq.as<int32_t>(), chunk, P->d_ent_need.as<int32_t>());
      RQB_CUDA(cudaGetLastError());
      std::vector<int32_t> need(P->ntasks);
      RQB_CUDA(cudaMemcpyAsync(need.data(), P->d_ent_need.p, sizeof(int32_t) * P->ntasks, cudaMemcpyDeviceToHost, fe.stream));
      RQB_CUDA(cudaStreamSynchronize(fe.stream));
      if (P->nready > 1) {
        std::stable_sort(q.begin(), q.end(), [&](int32_t a, int32_t b) { return need[a] < need[b]; });
        // feeder (see factor_dag_kernel): the initial tasks must be exactly the SMALL / ASM tasks of
        // the childless fronts, which is how the kernel recognises them
        const int kInitWindow = std::getenv("RQB_FEED_WINDOW") ? std::max(64, std::atoi(std::getenv("RQB_FEED_WINDOW"))) : 320;  // measured (e2e refactor, ms): 320 / 600 / 1024 / 2048 / 4096: cfg4_riga 26.6 / 26.7 / 26.9 / 27.3 / 27.3, cfg4_iga 60.7 / 61.0 / 61.4 / 62.7 / 63.7
        static const bool feed = !(std::getenv("RQB_FEED_INIT") && std::atoi(std::getenv("RQB_FEED_INIT")) == 0);
        int nleaf_tasks = 0;
        for (size_t t = 0; t < tasks.size(); ++t)
          nleaf_tasks += (tasks[t].type == T_SMALL || tasks[t].type == T_ASM) && S.fronts[tasks[t].front].children.empty();
        std::vector<int32_t> q0v(q);
        if (feed && P->nready > kInitWindow && nleaf_tasks == P->nready) {
          P->ninit = P->nready;
          P->d_init.upload(q.data(), sizeof(int32_t) * P->nready, fe.stream);
          std::fill(q0v.begin() + kInitWindow, q0v.end(), -1);
          const int qc[4] = {0, kInitWindow, kInitWindow, 0};
          RQB_CUDA(cudaMemcpyAsync(P->d_qctl0.p, qc, sizeof(qc), cudaMemcpyHostToDevice, fe.stream));
        }
        RQB_CUDA(cudaMemcpyAsync(P->d_queue0.p, q0v.data(), sizeof(int32_t) * P->nready, cudaMemcpyHostToDevice, fe.stream));
        RQB_CUDA(cudaStreamSynchronize(fe.stream));
      }
    }
    RQB_CUDA(cudaStreamSynchronize(fe.stream));  // the temporaries are freed on return
  }
  fe.dag_lazy = P->lazy != 0;
  P->dag_h = dag;
  fe.dag.reset(P.release());
}

// Evidence entry for the large-front Schur update: every UPDCB tile of ONE
// front (contribution block -= L21 U12, K = npiv, the DAG kernel's own
// updcb_task code) as a plain grid, so ncu's DMMA-pipe counters see the Schur
// update alone. Overwrites that front's contribution block (development use:
// refactor afterwards).
template <int kMinBlocks>
__global__ void __launch_bounds__(kDT, kMinBlocks) updcb_bench_kernel(double* pool, const FrontDev* fronts, int f,
                                                                     int acb, int tiles) {
  extern __shared__ double sm[];
  DagArgs A{};
  A.pool = pool;
  const FrontDev F = fronts[f];
  const int n = tiles - acb;
  for (int t = blockIdx.x; t < n * n; t += gridDim.x) {
    updcb_task(A, F, acb + t % n, acb + t / n, sm);
    __syncthreads();
  }
}

void rqb_dag_bench_updcb(FactorEngine& fe, int front, int reps, double* out) {
  if (!fe.dag) fail(errc::config, "the task-DAG factorization is not active");
  DagPlan& P = *fe.dag;
  const Symbolic& S = fe.sym;
  if (front < 0) {  // the front with the most contribution-block update flops
    double best = -1.0;
    for (int f = 0; f < static_cast<int>(S.fronts.size()); ++f) {
      const FrontDag& D = P.dag_h[f];
      if (D.acb >= D.tiles) continue;
      const double m = static_cast<double>(S.fronts[f].nf - D.acb * kTile);
      const double w = 2.0 * S.fronts[f].npiv * m * m;
      if (w > best) best = w, front = f;
    }
  }
  if (front < 0 || front >= static_cast<int>(S.fronts.size()) || P.dag_h[front].acb >= P.dag_h[front].tiles)
    fail(errc::config, "bench_updcb: the front has no contribution-block tiles");
  const FrontDag& D = P.dag_h[front];
  const int n = D.tiles - D.acb;
  auto kern = updcb_bench_kernel<2>;
  smem_at_least(kern, P.smem);
  int nsm = 148, occ = 1;
  RQB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, fe.device));
  RQB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kDT, P.smem));
  const int grid = std::max(1, std::min(n * n, nsm * std::max(1, occ)));
  kern<<<grid, kDT, P.smem, fe.stream>>>(fe.d_pool.as<double>(), fe.d_fronts.as<FrontDev>(), front, D.acb, D.tiles);
  RQB_CUDA(cudaGetLastError());
  RQB_CUDA(cudaEventRecord(fe.ev0, fe.stream));
  for (int r = 0; r < reps; ++r)
    kern<<<grid, kDT, P.smem, fe.stream>>>(fe.d_pool.as<double>(), fe.d_fronts.as<FrontDev>(), front, D.acb, D.tiles);
  RQB_CUDA(cudaEventRecord(fe.ev1, fe.stream));
  RQB_CUDA(cudaEventSynchronize(fe.ev1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, fe.ev0, fe.ev1);
  const double m = static_cast<double>(S.fronts[front].nf - D.acb * kTile);
  out[0] = ms / std::max(1, reps);
  out[1] = 2.0 * S.fronts[front].npiv * m * m;
  out[2] = front;
  out[3] = static_cast<double>(n) * n;
  out[4] = S.fronts[front].npiv;
  out[5] = grid;
}

void rqb_dag_enqueue(FactorEngine& fe) {
  DagPlan& P = *fe.dag;
  RQB_CUDA(cudaMemsetAsync(P.d_cnt.p, 0, P.d_cnt.bytes, fe.stream));
  RQB_CUDA(cudaMemsetAsync(P.d_tile.p, 0, P.d_tile.bytes, fe.stream));
  RQB_CUDA(cudaMemsetAsync(P.d_flagbits.p, 0, P.d_flagbits.bytes, fe.stream));
  RQB_CUDA(cudaMemcpyAsync(P.d_deps.p, P.d_deps0.p, P.d_deps0.bytes, cudaMemcpyDeviceToDevice, fe.stream));
  RQB_CUDA(cudaMemcpyAsync(P.d_queue.p, P.d_queue0.p, P.d_queue0.bytes, cudaMemcpyDeviceToDevice, fe.stream));
  RQB_CUDA(cudaMemcpyAsync(P.d_qctl.p, P.d_qctl0.p, P.d_qctl0.bytes, cudaMemcpyDeviceToDevice, fe.stream));
  DagArgs A;
  A.upd_cp16 = std::getenv("RQB_UPD_CP16") ? std::atoi(std::getenv("RQB_UPD_CP16")) : 1;
  A.upd_batch = P.upd_batch;
  A.rc_group = P.rc_group;
  A.upd_tma = std::getenv("RQB_UPD_TMA") ? std::atoi(std::getenv("RQB_UPD_TMA")) : 0;
  A.upd_la = P.upd_la;
  A.ubase = P.d_ubase.as<int32_t>();
  A.lazy = P.lazy;
  A.keep_small = std::getenv("RQB_KEEP_SMALL") ? std::atoi(std::getenv("RQB_KEEP_SMALL")) : 1;
  A.aval = fe.d_aval.as<double>();
  A.arrived = fe.d_arrived.as<int>();
  A.ent_need = P.d_ent_need.as<int32_t>();
  A.init_list = P.ninit > 0 ? P.d_init.as<int32_t>() : nullptr;
  A.ninit = P.ninit;
  A.ent_src = P.d_ent_src.as<int32_t>();
  A.ent_dst = P.d_ent_dst.as<int64_t>();
  A.ent_beg = P.d_ent_beg.as<int32_t>();
  A.ent_end = P.d_ent_end.as<int32_t>();
  A.fronts = fe.d_fronts.as<FrontDev>();
  A.dag = P.d_dag.as<FrontDag>();
  A.tasks = P.d_tasks.as<Task>();
  A.ntasks = P.ntasks;
  A.nqueued = P.nqueued;
  A.inv = fe.d_inv.as<int32_t>();
  A.rel = fe.d_rel.as<int32_t>();
  A.bnd = P.d_bnd.as<int32_t>();
  A.pool = fe.d_pool.as<double>();
  A.ipiv = fe.d_ipiv.as<int32_t>();
  A.scratch = fe.d_scratch.as<double>();
  A.backup = P.d_backup.as<double>();
  A.cnt = P.d_cnt.as<int>();
  A.tile_step = P.d_tile.as<int>();
  A.rc_prefix = P.d_rc.as<int32_t>();
  A.flagbits = P.d_flagbits.as<unsigned long long>();
  A.flags = fe.d_flags.as<int>();
  A.deps = P.d_deps.as<int>();
  A.queue = P.d_queue.as<int>();
  A.qctl = P.d_qctl.as<int>();
  A.step_base = P.d_sb.as<int32_t>();
  A.small_backup = P.d_small_backup.as<double>();
  A.prof = nullptr;
  A.trace = nullptr;
  if (fe.dag_prof_enabled) {
    if (!P.d_prof.p) P.d_prof.alloc(sizeof(unsigned long long) * 32);
    RQB_CUDA(cudaMemsetAsync(P.d_prof.p, 0, P.d_prof.bytes, fe.stream));
    A.prof = P.d_prof.as<unsigned long long>();
    if (std::getenv("RQB_DAG_TRACE")) {
      if (!P.d_trace.p) P.d_trace.alloc(sizeof(unsigned long long) * 4 * P.ntasks);
      A.trace = P.d_trace.as<unsigned long long>();
    }
  }
  A.small_nf = P.small_nf;
  smem_at_least(P.occ == 2 ? factor_dag_kernel<2> : factor_dag_kernel<1>, P.smem);
  if (P.occ == 2)
    factor_dag_kernel<2><<<P.grid, kDT, P.smem, fe.stream>>>(A);
  else
    factor_dag_kernel<1><<<P.grid, kDT, P.smem, fe.stream>>>(A);
  RQB_CUDA(cudaGetLastError());
}

// Per task type (SMALL, ASM, DIAG, ROWS, COLS, UPD): busy ms, wait ms (summed
// over CTAs, SM clock), count; plus the persistent grid size. Profiling run.
void rqb_dag_profile(FactorEngine& fe, double* out) {
  if (!fe.dag) fail(errc::config, "the task-DAG factorization is not active");
  fe.dag_prof_enabled = true;
  fe.enqueue_factor();
  fe.dag_prof_enabled = false;
  unsigned long long h[32];
  RQB_CUDA(cudaMemcpyAsync(h, fe.dag->d_prof.p, sizeof(h), cudaMemcpyDeviceToHost, fe.stream));
  RQB_CUDA(cudaStreamSynchronize(fe.stream));
  int clk_khz = 1965000;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, fe.device);
  for (int t = 0; t < 6; ++t) {
    out[3 * t + 0] = h[3 * t + 0] / (clk_khz * 1.0);  // cycles / kHz = ms
    out[3 * t + 1] = h[3 * t + 1] / (clk_khz * 1.0);
    out[3 * t + 2] = static_cast<double>(h[3 * t + 2]);
  }
  out[18] = fe.dag->grid;
  out[19] = fe.dag->ntasks;
  out[20] = h[20] / (clk_khz * 1.0);  // ready-queue pop wait, summed over CTAs
  out[21] = h[21] / (clk_khz * 1.0);  // UPDCB busy ms (UPD in slot 5 holds the per-step updates only)
  out[22] = 0;
  out[23] = static_cast<double>(h[23]);
  if (std::getenv("RQB_DAG_PROF_SMALL"))  // SMALL sub-phases, CTA-ms
    std::fprintf(stderr, "[dag] SMALL phases ms: assemble %.1f extend_add %.1f load %.1f panels %.1f writeback %.1f cb_update %.1f\n",
                 h[24] / (clk_khz * 1.0), h[25] / (clk_khz * 1.0), h[26] / (clk_khz * 1.0), h[27] / (clk_khz * 1.0),
                 h[28] / (clk_khz * 1.0), h[29] / (clk_khz * 1.0));
  if (const char* path = std::getenv("RQB_DAG_TRACE")) {  // development trace: tasks + timestamps
    DagPlan& P = *fe.dag;
    std::vector<unsigned long long> tr(4 * static_cast<size_t>(P.ntasks));
    std::vector<Task> tk(P.ntasks);
    RQB_CUDA(cudaMemcpy(tr.data(), P.d_trace.p, sizeof(unsigned long long) * tr.size(), cudaMemcpyDeviceToHost));
    RQB_CUDA(cudaMemcpy(tk.data(), P.d_tasks.p, sizeof(Task) * tk.size(), cudaMemcpyDeviceToHost));
    if (FILE* fp = std::fopen(path, "wb")) {
      const int32_t nt = P.ntasks;
      std::fwrite(&nt, sizeof(nt), 1, fp);
      std::fwrite(tk.data(), sizeof(Task), tk.size(), fp);
      std::fwrite(tr.data(), sizeof(unsigned long long), tr.size(), fp);
      std::fclose(fp);
    }
  }
}

// After a watchdog stall: the tasks whose dependency counters never reached
// zero (first few, in task order), for the error message.
std::string rqb_dag_stall_report(FactorEngine& fe) {
  DagPlan& P = *fe.dag;
  std::vector<int32_t> deps(P.ntasks);
  std::vector<Task> tk(P.ntasks);
  cudaMemcpy(deps.data(), P.d_deps.p, sizeof(int32_t) * P.ntasks, cudaMemcpyDeviceToHost);
  cudaMemcpy(tk.data(), P.d_tasks.p, sizeof(Task) * P.ntasks, cudaMemcpyDeviceToHost);
  static const char* names[] = {"SMALL", "ASM", "DIAG", "ROWS", "COLS", "UPD", "UPDCB", "UPDB"};
  std::string out;
  int shown = 0, pending = 0;
  for (int t = 0; t < P.ntasks; ++t) {
    if (deps[t] == 0 || (tk[t].type == T_DIAG && tk[t].step > 0)) continue;  // fused DIAGs are never counted down
    if (deps[t] >= (1 << 29)) continue;  // per-step update folded into an UPDB batch: never runs
    ++pending;
    if (shown < 6) {
      const Task& T = tk[t];
      out += std::string(shown ? ", " : "") + names[T.type] + "(front " + std::to_string(T.front) + ", step " +
             std::to_string(T.step) + ", " + std::to_string(T.a) + "," + std::to_string(T.b) + ") deps=" +
             std::to_string(deps[t]);
      ++shown;
    }
  }
  return std::to_string(pending) + " tasks never ready: " + out;
}

void DagPlanDeleter::operator()(DagPlan* p) const { delete p; }

}  // namespace rqb
