// SPDX-License-Identifier: Apache-2.0
// Multifrontal forward/backward substitution (solve_factored)
// as two persistent, sync-free kernels (one per sweep) over the device-resident
// fronts.
//
// Work items are 64-row blocks of a front (pivot blocks, then contribution
// rows), listed in a topological order of the dependency DAG (postorder of
// the elimination tree forward, its reverse backward). CTAs draw items with an
// atomic ticket, so an item only ever waits (spins) on items with smaller
// tickets that are already running: no inter-launch waits, no level barriers,
// and the whole sweep is one launch. Per item:
//   forward   w = b(pivot rows, after the front's net row permutation) +
//             children's contribution vectors (gather, atomic-free);
//             s = sum over finished pivot blocks j of L[rows, j] y_j
//             (left-looking, consumed as each block is published);
//             pivot block: unit-lower 64x64 triangle from shared memory, write
//             y, publish; contribution block: write w - s for the parent.
//   backward  s = y - U[rows, cb] x_cb (ancestors' solution, already final)
//             - U[rows, later pivot blocks] x (published in reverse order);
//             upper 64x64 triangle; write x (ND order for descendants, caller
//             order scaled, and the fused r_l = s r_u + v_u of apply_operator).
// Loads of data produced inside the sweep use ld.global.cg (L1 bypass);
// publication is __threadfence + atomicAdd, consumption volatile-spin +
// __threadfence.
#include <algorithm>

#include "device.cuh"

namespace rqb {

constexpr int kRB = 64;   // rows per item
constexpr int kST = 256;  // threads per CTA

struct SolveItem {
  int32_t front, r0, r1, blk;  // local rows [r0, r1), pivot-block index (-1: contribution rows)
};

__device__ __forceinline__ void wait_ge(const int* p, int target) {
  if (*((volatile const int*)p) >= target) return;
  while (*((volatile const int*)p) < target) __nanosleep(64);
}

__device__ __forceinline__ void publish(int* p) {
  __threadfence();
  atomicAdd(p, 1);
}

// cnt layout per front: [3f+0] pivot blocks published, [3f+1] items published,
// [3f+2] backward pivot blocks published. tickets: [0] fwd, [1] bwd.
__global__ void __launch_bounds__(kST) fwd_sweep(
    const FrontDev* __restrict__ fronts, const SolveItem* __restrict__ items, int nitems,
    const int32_t* __restrict__ nitems_front, const int32_t* __restrict__ inv,
    const double* __restrict__ pool, const int32_t* __restrict__ rowperm,
    const int32_t* __restrict__ perm, const double* __restrict__ b, double* __restrict__ y,
    double* __restrict__ cbvec, int* __restrict__ cnt, int* __restrict__ tickets) {
  __shared__ double D[kRB * (kRB + 1)];
  __shared__ double yb[kRB];
  __shared__ double part[4][kRB];
  __shared__ double wv[kRB];
  __shared__ int item_s;
  const int tid = threadIdx.x, row = tid & (kRB - 1), grp = tid >> 6;
  for (;;) {
    __syncthreads();
    if (tid == 0) item_s = atomicAdd(&tickets[0], 1);
    __syncthreads();
    const int it = item_s;
    if (it >= nitems) return;
    const SolveItem I = items[it];
    const FrontDev F = fronts[I.front];
    const int np = F.npiv, nr = I.r1 - I.r0;
    const double* g = pool + F.off;
    const int64_t ld = F.ld;
    // (1) everything that does not depend on other items: index maps, b, the
    //     diagonal block, the first L block of this thread
    const int32_t* inv0 = inv + F.inv_off;
    double bv = 0.0;
    int ir0 = -1, ir1 = -1;
    if (tid < nr) {
      const int r = I.r0 + tid;
      const int q = r < np ? __ldg(&rowperm[F.start + r]) : r;  // pre-swap local row
      bv = q < np ? b[perm[F.start + q]] : 0.0;
      if (F.nchild > 0) ir0 = inv0[q];
      if (F.nchild > 1) ir1 = inv0[F.nf + q];
    }
    if (I.blk >= 0)
      for (int idx = tid; idx < nr * nr; idx += kST) {
        const int r = idx % nr, c = idx / nr;
        D[r + c * (kRB + 1)] = g[(I.r0 + r) + (int64_t)(I.r0 + c) * ld];
      }
    const int nblk = I.blk >= 0 ? I.blk : (np + kRB - 1) / kRB;
    double lreg[kRB / 4];
    auto prefetch = [&](int j) {
      const int c0 = j * kRB, cw = min(np, c0 + kRB) - c0;
      const double* lp = g + (I.r0 + row) + (int64_t)c0 * ld;
#pragma unroll
      for (int u = 0; u < kRB / 4; ++u) {
        const int c = grp + 4 * u;
        lreg[u] = (row < nr && c < cw) ? lp[c * ld] : 0.0;
      }
    };
    if (nblk > 0) prefetch(0);
    // (2) children complete -> gather their contribution vectors
    if (tid == 0) {
      if (F.nchild > 0) wait_ge(&cnt[3 * F.child0 + 1], nitems_front[F.child0]);
      if (F.nchild > 1) wait_ge(&cnt[3 * F.child1 + 1], nitems_front[F.child1]);
      __threadfence();
    }
    __syncthreads();
    if (tid < nr) {
      double v = bv;
      if (ir0 >= 0) v += __ldcg(&cbvec[fronts[F.child0].cbvec_off + ir0 - fronts[F.child0].npiv]);
      if (ir1 >= 0) v += __ldcg(&cbvec[fronts[F.child1].cbvec_off + ir1 - fronts[F.child1].npiv]);
      wv[tid] = v;
    }
    // (3) left-looking over the published pivot blocks, next L block prefetched
    double s = 0.0;
    for (int j = 0; j < nblk; ++j) {
      if (tid == 0) {
        wait_ge(&cnt[3 * I.front + 0], j + 1);
        __threadfence();
      }
      __syncthreads();
      const int c0 = j * kRB, c1 = min(np, c0 + kRB);
      if (tid < kRB) yb[tid] = tid < c1 - c0 ? __ldcg(&y[F.start + c0 + tid]) : 0.0;
      __syncthreads();
#pragma unroll
      for (int u = 0; u < kRB / 4; ++u) s += lreg[u] * yb[grp + 4 * u];
      if (j + 1 < nblk) prefetch(j + 1);
    }
    part[grp][row] = s;
    __syncthreads();
    if (tid < nr) wv[tid] -= part[0][tid] + part[1][tid] + part[2][tid] + part[3][tid];
    if (I.blk >= 0) {
      // unit-lower diagonal block (already in shared memory)
      __syncthreads();
      if (tid < 32) {
        double v0 = tid < nr ? wv[tid] : 0.0, v1 = tid + 32 < nr ? wv[tid + 32] : 0.0;
        for (int c = 0; c < nr; ++c) {
          const double yc = c < 32 ? __shfl_sync(0xffffffffu, v0, c) : __shfl_sync(0xffffffffu, v1, c - 32);
          if (tid > c) v0 -= D[tid + c * (kRB + 1)] * yc;
          if (tid + 32 > c && tid + 32 < nr) v1 -= D[tid + 32 + c * (kRB + 1)] * yc;
        }
        if (tid < nr) y[F.start + I.r0 + tid] = v0;
        if (tid + 32 < nr) y[F.start + I.r0 + tid + 32] = v1;
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(&cnt[3 * I.front + 0], 1);
        atomicAdd(&cnt[3 * I.front + 1], 1);
      }
    } else {
      if (tid < nr) cbvec[F.cbvec_off + I.r0 + tid - np] = wv[tid];
      __syncthreads();
      if (tid == 0) publish(&cnt[3 * I.front + 1]);
    }
  }
}

__global__ void __launch_bounds__(kST) bwd_sweep(
    const FrontDev* __restrict__ fronts, const SolveItem* __restrict__ items, int nitems,
    const int32_t* __restrict__ npb_front, const int32_t* __restrict__ parent,
    const int32_t* __restrict__ rows, const double* __restrict__ pool,
    const int32_t* __restrict__ perm, const double* __restrict__ y, double* __restrict__ xnew,
    double* __restrict__ xout, double scale, const double* __restrict__ vu, double sigma,
    double* __restrict__ xl_out, int* __restrict__ cnt, int* __restrict__ tickets) {
  __shared__ double D[kRB * (kRB + 1)];
  __shared__ double xb[kRB];
  __shared__ double part[4][kRB];
  __shared__ int item_s;
  const int tid = threadIdx.x, row = tid & (kRB - 1), grp = tid >> 6;
  for (;;) {
    __syncthreads();
    if (tid == 0) item_s = atomicAdd(&tickets[1], 1);
    __syncthreads();
    const int it = item_s;
    if (it >= nitems) return;
    const SolveItem I = items[it];
    const FrontDev F = fronts[I.front];
    const int np = F.npiv, nf = F.nf, nr = I.r1 - I.r0;
    const int par = parent[I.front];
    const double* g = pool + F.off;
    const int64_t ld = F.ld;
    const int32_t* rw = rows + F.rows_off;
    // (1) independent loads: diagonal block, y of this block, first U chunk
    for (int idx = tid; idx < nr * nr; idx += kST) {
      const int r = idx % nr, c = idx / nr;
      D[r + c * (kRB + 1)] = g[(I.r0 + r) + (int64_t)(I.r0 + c) * ld];
    }
    double y0 = 0.0, y1 = 0.0;
    if (tid < 32) {
      if (tid < nr) y0 = y[F.start + I.r0 + tid];
      if (tid + 32 < nr) y1 = y[F.start + I.r0 + tid + 32];
    }
    const int npb = (np + kRB - 1) / kRB;
    const int ncbc = (nf - np + kRB - 1) / kRB;  // contribution-column chunks (ancestors' x)
    const int nch = ncbc + (npb - 1 - I.blk);     // + later pivot blocks (last first)
    auto chunk = [&](int t, int& c0, int& c1, bool& piv) {
      if (t < ncbc) {
        c0 = np + t * kRB;
        c1 = min(nf, c0 + kRB);
        piv = false;
      } else {
        const int j = npb - 1 - (t - ncbc);
        c0 = j * kRB;
        c1 = min(np, c0 + kRB);
        piv = true;
      }
    };
    double ureg[kRB / 4];
    auto prefetch = [&](int t) {
      int c0, c1;
      bool pv;
      chunk(t, c0, c1, pv);
      const double* up = g + (I.r0 + row) + (int64_t)c0 * ld;
#pragma unroll
      for (int u = 0; u < kRB / 4; ++u) {
        const int c = grp + 4 * u;
        ureg[u] = (row < nr && c < c1 - c0) ? up[c * ld] : 0.0;
      }
    };
    if (nch > 0) prefetch(0);
    if (tid == 0) {
      if (par >= 0) wait_ge(&cnt[3 * par + 2], npb_front[par]);
      __threadfence();
    }
    __syncthreads();
    double s = 0.0;
    for (int t = 0; t < nch; ++t) {
      int c0, c1;
      bool pv;
      chunk(t, c0, c1, pv);
      if (pv && tid == 0) {
        wait_ge(&cnt[3 * I.front + 2], npb - c0 / kRB);
        __threadfence();
      }
      __syncthreads();
      if (tid < kRB)
        xb[tid] = tid < c1 - c0 ? __ldcg(&xnew[pv ? F.start + c0 + tid : rw[c0 + tid]]) : 0.0;
      __syncthreads();
#pragma unroll
      for (int u = 0; u < kRB / 4; ++u) s += ureg[u] * xb[grp + 4 * u];
      if (t + 1 < nch) prefetch(t + 1);
    }
    part[grp][row] = s;
    __syncthreads();
    if (tid < 32) {
      double v0 = 0.0, v1 = 0.0;
      if (tid < nr) v0 = y0 - (part[0][tid] + part[1][tid] + part[2][tid] + part[3][tid]);
      if (tid + 32 < nr)
        v1 = y1 - (part[0][tid + 32] + part[1][tid + 32] + part[2][tid + 32] + part[3][tid + 32]);
      for (int c = nr - 1; c >= 0; --c) {
        if (c < 32) {
          if (tid == c) v0 /= D[c + c * (kRB + 1)];
        } else {
          if (tid == c - 32) v1 /= D[c + c * (kRB + 1)];
        }
        const double xc = c < 32 ? __shfl_sync(0xffffffffu, v0, c) : __shfl_sync(0xffffffffu, v1, c - 32);
        if (tid < c) v0 -= D[tid + c * (kRB + 1)] * xc;
        if (tid + 32 < c) v1 -= D[tid + 32 + c * (kRB + 1)] * xc;
      }
      for (int h = 0; h < 2; ++h) {
        const int r = tid + 32 * h;
        if (r < nr) {
          const double v = h ? v1 : v0;
          const int gi = F.start + I.r0 + r;
          xnew[gi] = v;
          const int o = perm[gi];
          const double sv = scale * v;
          xout[o] = sv;
          if (xl_out) xl_out[o] = sigma * sv + vu[o];
        }
      }
    }
    __syncthreads();
    if (tid == 0) publish(&cnt[3 * I.front + 2]);
  }
}

// Net row permutation of every front's pivot block after factorization:
// rowperm[start + k] = pre-swap local row found at position k.
__global__ void net_rowperm(const FrontDev* __restrict__ fronts, int nfronts,
                            const int32_t* __restrict__ ipiv, int32_t* __restrict__ rowperm) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nfronts) return;
  const FrontDev F = fronts[f];
  int32_t* rp = rowperm + F.start;
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

void FactorEngine::solve_device(const double* b, double* x, double scale_out) {
  rqb_solve_enqueue(*this, b, x, scale_out, nullptr, 0.0, nullptr);
}

void rqb_solve_prepare(FactorEngine& fe) {
  const Symbolic& S = fe.sym;
  const int nfr = static_cast<int>(S.fronts.size());
  std::vector<SolveItem> fwd, bwd;
  std::vector<int32_t> nitems(nfr, 0), npb(nfr, 0), parent(nfr, -1);
  for (int f = 0; f < nfr; ++f) {
    const Front& F = S.fronts[f];
    int a = F.parent;  // nearest ancestor that has pivots (empty separators pass through)
    while (a >= 0 && S.fronts[a].npiv == 0) a = S.fronts[a].parent;
    parent[f] = a;
    const int nb = (F.npiv + kRB - 1) / kRB;
    npb[f] = nb;
    for (int b = 0; b < nb; ++b) fwd.push_back({f, b * kRB, std::min(F.npiv, (b + 1) * kRB), b});
    for (int r = F.npiv; r < F.nf; r += kRB) fwd.push_back({f, r, std::min(F.nf, r + kRB), -1});
    nitems[f] = nb + (F.nf - F.npiv + kRB - 1) / kRB;
  }
  for (int f = nfr - 1; f >= 0; --f) {
    const Front& F = S.fronts[f];
    for (int b = npb[f] - 1; b >= 0; --b) bwd.push_back({f, b * kRB, std::min(F.npiv, (b + 1) * kRB), b});
  }
  fe.n_fwd_items = static_cast<int>(fwd.size());
  fe.n_bwd_items = static_cast<int>(bwd.size());
  if (fwd.empty()) fwd.push_back({0, 0, 0, -1});
  if (bwd.empty()) bwd.push_back({0, 0, 0, -1});
  fe.d_items_fwd.upload(fwd.data(), sizeof(SolveItem) * fwd.size(), fe.stream);
  fe.d_items_bwd.upload(bwd.data(), sizeof(SolveItem) * bwd.size(), fe.stream);
  fe.d_nitems.upload(nitems.data(), sizeof(int32_t) * nfr, fe.stream);
  fe.d_npb.upload(npb.data(), sizeof(int32_t) * nfr, fe.stream);
  fe.d_parent.upload(parent.data(), sizeof(int32_t) * nfr, fe.stream);
  fe.d_cnt.alloc(sizeof(int) * (3 * nfr + 8));
  fe.d_rowperm.alloc(sizeof(int32_t) * std::max<int64_t>(1, fe.n));
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, fe.device);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fwd_sweep, kST, 0);
  fe.solve_grid = std::max(1, nsm * std::max(1, occ));
}

void rqb_rowperm_enqueue(FactorEngine& fe) {
  const int nfr = static_cast<int>(fe.fronts_h.size());
  net_rowperm<<<(nfr + 127) / 128, 128, 0, fe.stream>>>(fe.d_fronts.as<FrontDev>(), nfr,
                                                        fe.d_ipiv.as<int32_t>(), fe.d_rowperm.as<int32_t>());
}

void rqb_solve_enqueue(FactorEngine& fe, const double* b, double* x, double scale, const double* vu,
                       double sigma, double* xl) {
  const int nfr = static_cast<int>(fe.fronts_h.size());
  RQB_CUDA(cudaMemsetAsync(fe.d_cnt.p, 0, sizeof(int) * (3 * nfr + 8), fe.stream));
  int* cnt = fe.d_cnt.as<int>();
  int* tickets = cnt + 3 * nfr;
  const int gf = std::min(fe.solve_grid, std::max(1, fe.n_fwd_items));
  fwd_sweep<<<gf, kST, 0, fe.stream>>>(
      fe.d_fronts.as<FrontDev>(), fe.d_items_fwd.as<SolveItem>(), fe.n_fwd_items, fe.d_nitems.as<int32_t>(),
      fe.d_inv.as<int32_t>(), fe.d_pool.as<double>(), fe.d_rowperm.as<int32_t>(), fe.d_perm.as<int32_t>(), b,
      fe.d_y.as<double>(), fe.d_cbvec.as<double>(), cnt, tickets);
  const int gb = std::min(fe.solve_grid, std::max(1, fe.n_bwd_items));
  bwd_sweep<<<gb, kST, 0, fe.stream>>>(
      fe.d_fronts.as<FrontDev>(), fe.d_items_bwd.as<SolveItem>(), fe.n_bwd_items, fe.d_npb.as<int32_t>(),
      fe.d_parent.as<int32_t>(), fe.d_rows.as<int32_t>(), fe.d_pool.as<double>(), fe.d_perm.as<int32_t>(),
      fe.d_y.as<double>(), fe.d_xnew.as<double>(), x, scale, vu, sigma, xl, cnt, tickets);
  RQB_CUDA(cudaGetLastError());
  fe.launches_solve = 2;
}

void rqb_solve_set_attrs(int) {}

}  // namespace rqb
