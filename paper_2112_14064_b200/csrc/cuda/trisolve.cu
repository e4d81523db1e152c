// SPDX-License-Identifier: Apache-2.0
// Multifrontal forward/backward substitution (solve_factored)
// over the device-resident fronts, level by level (leaves first forward, root
// first backward).
//
// Forward, per front (one CTA): w = [b(pivot rows); 0] + extend-add of the
// children's contribution vectors (gather, atomic-free), the front's row swaps,
// blocked unit-lower substitution over all nf rows (32-column blocks: the
// diagonal block in one warp with shuffles, the rows below as a GEMV whose
// column reads are coalesced), pivots -> y, remaining rows -> the front's
// contribution vector for the parent.
// Backward, per front: x_piv = U11^{-1} (y_piv - U12 x_cb), x_cb gathered from
// the ancestors' solution; writes the solution in ND order (for descendants)
// and, scaled, in the caller's ordering; optionally fuses r_l = s r_u + v_u of
// apply_operator.
#include "device.cuh"

namespace rqb {

template <int NT>
__global__ void __launch_bounds__(NT) fwd_level(const FrontDev* __restrict__ fronts,
                                               const int32_t* __restrict__ list,
                                               const int32_t* __restrict__ inv,
                                               const double* __restrict__ pool,
                                               const int32_t* __restrict__ ipiv,
                                               const int32_t* __restrict__ perm,
                                               const double* __restrict__ b,
                                               double* __restrict__ y, double* __restrict__ cbvec) {
  extern __shared__ double w[];
  const FrontDev F = fronts[list[blockIdx.x]];
  const int nf = F.nf, np = F.npiv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t* inv0 = inv + F.inv_off;
  const int32_t* inv1 = inv0 + nf;
  int c0off = 0, c0np = 0, c1off = 0, c1np = 0;
  if (F.nchild > 0) {
    c0off = (int)fronts[F.child0].cbvec_off;
    c0np = fronts[F.child0].npiv;
  }
  if (F.nchild > 1) {
    c1off = (int)fronts[F.child1].cbvec_off;
    c1np = fronts[F.child1].npiv;
  }
  for (int r = tid; r < nf; r += NT) {
    double v = r < np ? b[perm[F.start + r]] : 0.0;
    if (F.nchild > 0) {
      const int ir = inv0[r];
      if (ir >= 0) v += cbvec[c0off + ir - c0np];
    }
    if (F.nchild > 1) {
      const int ir = inv1[r];
      if (ir >= 0) v += cbvec[c1off + ir - c1np];
    }
    w[r] = v;
  }
  __syncthreads();
  if (tid == 0)
    for (int k = 0; k < np; ++k) {
      const int p = ipiv[F.start + k];
      if (p != k) {
        const double t = w[k];
        w[k] = w[p];
        w[p] = t;
      }
    }
  __syncthreads();
  const double* g = pool + F.off;
  const int64_t ld = F.ld;
  for (int kb = 0; kb < np; kb += 32) {
    const int bw = min(32, np - kb);
    if (warp == 0) {
      double wi = lane < bw ? w[kb + lane] : 0.0;
      for (int t = 0; t < bw; ++t) {
        const double yt = __shfl_sync(0xffffffffu, wi, t);
        if (lane > t && lane < bw) wi -= g[(kb + lane) + (kb + t) * ld] * yt;
      }
      if (lane < bw) w[kb + lane] = wi;
    }
    __syncthreads();
    for (int r = kb + bw + tid; r < nf; r += NT) {
      double s = 0.0;
      for (int t = 0; t < bw; ++t) s += g[r + (kb + t) * ld] * w[kb + t];
      w[r] -= s;
    }
    __syncthreads();
  }
  for (int r = tid; r < nf; r += NT) {
    if (r < np)
      y[F.start + r] = w[r];
    else
      cbvec[F.cbvec_off + r - np] = w[r];
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) bwd_level(const FrontDev* __restrict__ fronts,
                                               const int32_t* __restrict__ list,
                                               const int32_t* __restrict__ rows,
                                               const double* __restrict__ pool,
                                               const int32_t* __restrict__ perm,
                                               const double* __restrict__ y,
                                               double* __restrict__ xnew, double* __restrict__ xout,
                                               double scale, const double* __restrict__ vu,
                                               double sigma, double* __restrict__ xl_out) {
  extern __shared__ double x[];
  const FrontDev F = fronts[list[blockIdx.x]];
  const int nf = F.nf, np = F.npiv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t* rw = rows + F.rows_off;
  for (int r = tid; r < nf; r += NT) x[r] = r < np ? y[F.start + r] : xnew[rw[r]];
  __syncthreads();
  const double* g = pool + F.off;
  const int64_t ld = F.ld;
  for (int i = tid; i < np; i += NT) {
    double s = 0.0;
    for (int c = np; c < nf; ++c) s += g[i + c * ld] * x[c];
    x[i] -= s;
  }
  __syncthreads();
  for (int kb = ((np - 1) / 32) * 32; kb >= 0 && np > 0; kb -= 32) {
    const int bw = min(32, np - kb);
    if (warp == 0) {
      double xi = lane < bw ? x[kb + lane] : 0.0;
      for (int t = bw - 1; t >= 0; --t) {
        if (lane == t) xi /= g[(kb + t) + (kb + t) * ld];
        const double xt = __shfl_sync(0xffffffffu, xi, t);
        if (lane < t) xi -= g[(kb + lane) + (kb + t) * ld] * xt;
      }
      if (lane < bw) x[kb + lane] = xi;
    }
    __syncthreads();
    for (int r = tid; r < kb; r += NT) {
      double s = 0.0;
      for (int t = 0; t < bw; ++t) s += g[r + (kb + t) * ld] * x[kb + t];
      x[r] -= s;
    }
    __syncthreads();
  }
  for (int r = tid; r < np; r += NT) {
    const double v = x[r];
    xnew[F.start + r] = v;
    const int o = perm[F.start + r];
    const double sv = scale * v;
    xout[o] = sv;
    if (xl_out) xl_out[o] = sigma * sv + vu[o];
  }
}

namespace {
int div_up_i(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }
}  // namespace

void FactorEngine::solve_device(const double* b, double* x, double scale_out) {
  rqb_solve_enqueue(*this, b, x, scale_out, nullptr, 0.0, nullptr);
}

void rqb_solve_enqueue(FactorEngine& fe, const double* b, double* x, double scale, const double* vu,
                       double sigma, double* xl) {
  const FrontDev* fr = fe.d_fronts.as<FrontDev>();
  const int32_t* lists = fe.d_lists.as<int32_t>();
  const int32_t* perm = fe.d_perm.as<int32_t>();
  int64_t launches = 0;
  for (const LevelPlan& P : fe.plans) {
    const size_t smem = sizeof(double) * std::max(1, P.solve_maxnf);
    fwd_level<256><<<static_cast<unsigned>(P.all.size()), 256, smem, fe.stream>>>(
        fr, lists + P.off_all, fe.d_inv.as<int32_t>(), fe.d_pool.as<double>(),
        fe.d_ipiv.as<int32_t>(), perm, b, fe.d_y.as<double>(), fe.d_cbvec.as<double>());
    ++launches;
  }
  for (auto it = fe.plans.rbegin(); it != fe.plans.rend(); ++it) {
    const LevelPlan& P = *it;
    const size_t smem = sizeof(double) * std::max(1, P.solve_maxnf);
    bwd_level<256><<<static_cast<unsigned>(P.all.size()), 256, smem, fe.stream>>>(
        fr, lists + P.off_all, fe.d_rows.as<int32_t>(), fe.d_pool.as<double>(), perm,
        fe.d_y.as<double>(), fe.d_xnew.as<double>(), x, scale, vu, sigma, xl);
    ++launches;
  }
  RQB_CUDA(cudaGetLastError());
  fe.launches_solve = launches;
}

void rqb_solve_set_attrs(int maxnf) {
  const int smem = sizeof(double) * maxnf;
  if (smem > 48 * 1024) {
    RQB_CUDA(cudaFuncSetAttribute(fwd_level<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    RQB_CUDA(cudaFuncSetAttribute(bwd_level<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
}

}  // namespace rqb
