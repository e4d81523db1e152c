// SPDX-License-Identifier: Apache-2.0
// Device assembly of the BASELINE pencil (the host
// assembler is csrc/host/spaces.cpp:assemble_pencil, SPEC.md:216-224,
// 261-264 for the forms / quadrature / elimination rules).
//
// Produces the same CSR pattern and the same K, C, M values bit for bit:
//   1. pattern: per free row, the free DOFs of both components whose support
//      boxes overlap the row's (count kernel, device scan, warp-per-row fill
//      with ballot compaction, same sorted order as the host).
//   2. element matrices: one CTA per element computes the upper triangle of
//      the local K and M over the (p+1)^2 Gauss points in the host's order
//      (qy outer, qx inner) with every product and sum rounded separately
//      (__dmul_rn / __dadd_rn; the host file is built with -ffp-contract=off).
//   3. gather: one warp per row; each nnz entry sums its element
//      contributions in the order the host scatters them — element-row colour
//      ey mod (p+1) ascending, then ex ascending — so the global sums round
//      identically, with no atomics (deterministic).
// The element matrices stay in HBM between stages 2 and 3 (2 x ne^2 x
// nloc(nloc+1)/2 doubles: 1.3 GB at cfg4).
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cstring>

#include "device.cuh"

namespace rqb {

namespace {

struct AsmArgs {
  int ne, nq, kind_curl, stride;
  int nloc, ntri, locsz0;
  int px[2], py[2];        // degrees of component c in x / y
  int nbx[2], nby[2];      // basis counts
  int64_t base[2];         // first full id of component c
  int64_t n;               // free DOFs
  const int32_t* f2f;      // full -> free (-1 constrained)
  const int32_t* free2full;
  const int32_t* box;      // 4 per free DOF
  // per component c, direction d: first basis of element e, support ranges
  const int32_t* first[2][2];
  const int32_t* supf[2][2];
  const int32_t* supl[2][2];
  const double* val[2][2];  // [e][q][a]
  const double* der[2][2];
  const double* w[2];       // weights of component 0, direction d: [e][q]
  const int32_t* pairs;     // packed upper triangle (r | s << 16), ntri
  double* Kel;              // [e][ntri]
  double* Mel;
};

// first basis a with sup_last[a] >= lo (sup_last nondecreasing)
__device__ __forceinline__ int lower_sup(const int32_t* supl, int nb, int lo) {
  int a = 0, b = nb;
  while (a < b) {
    const int m = (a + b) >> 1;
    if (supl[m] < lo) a = m + 1; else b = m;
  }
  return a;
}
// last basis b with sup_first[b] <= hi (sup_first nondecreasing)
__device__ __forceinline__ int upper_sup(const int32_t* supf, int nb, int hi) {
  int a = 0, b = nb;
  while (a < b) {
    const int m = (a + b) >> 1;
    if (supf[m] <= hi) a = m + 1; else b = m;
  }
  return a - 1;
}

struct RowRange {
  int i0[2], i1[2], j0[2], j1[2];
};

__device__ __forceinline__ RowRange row_range(const AsmArgs& A, int64_t r) {
  const int32_t* b = A.box + 4 * r;
  RowRange R;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    R.i0[c] = lower_sup(A.supl[c][0], A.nbx[c], b[0]);
    R.i1[c] = upper_sup(A.supf[c][0], A.nbx[c], b[1]);
    R.j0[c] = lower_sup(A.supl[c][1], A.nby[c], b[2]);
    R.j1[c] = upper_sup(A.supf[c][1], A.nby[c], b[3]);
  }
  return R;
}

__global__ void asm_count(AsmArgs A, int64_t* counts) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= A.n) return;
  const RowRange R = row_range(A, r);
  int64_t cnt = 0;
  for (int c = 0; c < 2; ++c)
    for (int j = R.j0[c]; j <= R.j1[c]; ++j) {
      const int32_t* f = A.f2f + A.base[c] + static_cast<int64_t>(j) * A.nbx[c];
      for (int i = R.i0[c]; i <= R.i1[c]; ++i) cnt += f[i] >= 0;
    }
  counts[r] = cnt;
}

__global__ void asm_fill(AsmArgs A, const int64_t* rowptr, int32_t* col) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); r < A.n;
       r += nwarps) {
    const RowRange R = row_range(A, r);
    int64_t pos = rowptr[r];
    // the (j, i) box of each component flattened j-major: lanes cover whole
    // box rows at once, and the flattened order is the sorted column order
    for (int c = 0; c < 2; ++c) {
      const int w = R.i1[c] - R.i0[c] + 1, h = R.j1[c] - R.j0[c] + 1;
      if (w <= 0 || h <= 0) continue;
      const int32_t* f = A.f2f + A.base[c] + static_cast<int64_t>(R.j0[c]) * A.nbx[c] + R.i0[c];
      for (int t0 = 0; t0 < w * h; t0 += 32) {
        const int t = t0 + lane;
        int32_t v = -1;
        if (t < w * h) {
          const int jj = t / w;
          v = f[static_cast<int64_t>(jj) * A.nbx[c] + (t - jj * w)];
        }
        const unsigned m = __ballot_sync(0xffffffffu, v >= 0);
        if (v >= 0) col[pos + __popc(m & ((1u << lane) - 1u))] = v;
        pos += __popc(m);
      }
    }
  }
}

// Element matrices: CTA per element, Gauss points staged in shared memory in
// chunks of `rows` qy-lines; partial sums carried across chunks through the
// output (exact: doubles in, doubles out).
__global__ void asm_element(AsmArgs A, int rows) {
  extern __shared__ double sm[];  // [rows*nq] weights, then [pt][o][2] values
  const int e = blockIdx.x;
  const int ex = e % A.ne, ey = e / A.ne;
  const int nq = A.nq, nloc = A.nloc;
  double* sw = sm;
  double* sv = sm + ((rows * nq + 1) & ~1);
  double* Ke = A.Kel + static_cast<int64_t>(e) * A.ntri;
  double* Me = A.Mel + static_cast<int64_t>(e) * A.ntri;
  for (int qy0 = 0; qy0 < nq; qy0 += rows) {
    const int ny = min(rows, nq - qy0), npt = ny * nq;
    for (int t = threadIdx.x; t < npt * nloc; t += blockDim.x) {
      const int pt = t / nloc, o = t - pt * nloc;
      const int qy = qy0 + pt / nq, qx = pt % nq;
      const int c = o < A.locsz0 ? 0 : 1;
      const int oo = o - (c ? A.locsz0 : 0);
      const int a = oo % (A.px[c] + 1), b = oo / (A.px[c] + 1);
      const int64_t ox = (static_cast<int64_t>(ex) * nq + qx) * (A.px[c] + 1) + a;
      const int64_t oy = (static_cast<int64_t>(ey) * nq + qy) * (A.py[c] + 1) + b;
      const double vx = A.val[c][0][ox], dx = A.der[c][0][ox];
      const double vy = A.val[c][1][oy], dy = A.der[c][1][oy];
      double dd;
      if (!A.kind_curl)
        dd = c == 0 ? __dmul_rn(dx, vy) : __dmul_rn(vx, dy);  // div
      else
        dd = c == 0 ? -__dmul_rn(vx, dy) : __dmul_rn(dx, vy);  // curl
      sv[2 * t] = __dmul_rn(vx, vy);
      sv[2 * t + 1] = dd;
      if (o == 0)
        sw[pt] = __dmul_rn(A.w[0][static_cast<int64_t>(ex) * nq + qx],
                           A.w[1][static_cast<int64_t>(ey) * nq + qy]);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < A.ntri; t += blockDim.x) {
      const int32_t pr = A.pairs[t];
      const int r = pr & 0xffff, s = pr >> 16;
      const bool same = (r < A.locsz0) == (s < A.locsz0);
      double k = qy0 ? Ke[t] : 0.0, m = qy0 ? Me[t] : 0.0;
      for (int pt = 0; pt < npt; ++pt) {
        const double w = sw[pt];
        const double* v = sv + 2 * pt * nloc;
        const double vr = __dmul_rn(w, v[2 * r]), dr = __dmul_rn(w, v[2 * r + 1]);
        const double mm = same ? __dmul_rn(vr, v[2 * s]) : 0.0;
        k = __dadd_rn(k, __dadd_rn(__dmul_rn(dr, v[2 * s + 1]), mm));
        m = __dadd_rn(m, mm);
      }
      Ke[t] = k;
      Me[t] = m;
    }
    __syncthreads();
  }
}

struct DofInfo {
  int c, i, j;
};
__device__ __forceinline__ DofInfo dof_info(const AsmArgs& A, int64_t f) {
  const int64_t g = A.free2full[f];
  DofInfo d;
  d.c = g >= A.base[1] ? 1 : 0;
  const int64_t l = g - A.base[d.c];
  d.i = static_cast<int>(l % A.nbx[d.c]);
  d.j = static_cast<int>(l / A.nbx[d.c]);
  return d;
}
__device__ __forceinline__ int local_index(const AsmArgs& A, const DofInfo& d, int ex, int ey) {
  const int a = d.i - A.first[d.c][0][ex], b = d.j - A.first[d.c][1][ey];
  return (d.c ? A.locsz0 : 0) + b * (A.px[d.c] + 1) + a;
}

__global__ void asm_gather(AsmArgs A, const int64_t* rowptr, const int32_t* col, double alpha,
                           double beta, double* K, double* C, double* M) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); r < A.n;
       r += nwarps) {
    const DofInfo dr = dof_info(A, r);
    const int4 br = *reinterpret_cast<const int4*>(A.box + 4 * r);
    for (int64_t k = rowptr[r] + lane; k < rowptr[r + 1]; k += 32) {
      const int32_t s = col[k];
      const DofInfo ds = dof_info(A, s);
      const int4 bs = *reinterpret_cast<const int4*>(A.box + 4 * static_cast<int64_t>(s));
      const int ex0 = max(br.x, bs.x), ex1 = min(br.y, bs.y);
      const int ey0 = max(br.z, bs.z), ey1 = min(br.w, bs.w);
      double kv = 0.0, mv = 0.0;
      for (int cy = 0; cy < A.stride; ++cy) {
        const int ey = ey0 + (cy - ey0 % A.stride + A.stride) % A.stride;
        if (ey > ey1) continue;
        for (int ex = ex0; ex <= ex1; ++ex) {
          const int lr = local_index(A, dr, ex, ey), ls = local_index(A, ds, ex, ey);
          const int lo = min(lr, ls), hi = max(lr, ls);
          const int64_t idx = static_cast<int64_t>(ey * A.ne + ex) * A.ntri +
                              (lo * A.nloc - lo * (lo - 1) / 2 + hi - lo);
          kv = __dadd_rn(kv, A.Kel[idx]);
          mv = __dadd_rn(mv, A.Mel[idx]);
        }
      }
      K[k] = kv;
      M[k] = mv;
      C[k] = __dadd_rn(__dmul_rn(alpha, mv), __dmul_rn(beta, kv));
    }
  }
}

}  // namespace

Pencil assemble_pencil_device(const VectorSpace& vs, double alpha, double beta, double* ms,
                              DevicePencil* keep) {
  if (vs.degree > kMaxAsmDegree) fail(errc::domain, "degree too large for assembly tables");
  Pencil P;
  P.elems = vs.elems;
  P.n_full = vs.N();
  if (P.n_full >= (int64_t(1) << 31)) fail(errc::config, "device assembly: more than 2^31 DOFs");
  using clk = std::chrono::steady_clock;
  const auto t_host0 = clk::now();
  std::vector<int64_t> full_to_free;
  free_numbering(vs, &full_to_free, &P.free_to_full);
  P.n = static_cast<int64_t>(P.free_to_full.size());
  P.box = support_boxes(vs, P.free_to_full);
  QuadTable tab[2][2];
  quad_tables(vs, tab);
  const Tensor2* comp[2] = {&vs.cx, &vs.cy};
  const int ne = vs.elems, nq = vs.degree + 1;

  AsmArgs A{};
  A.ne = ne;
  A.nq = nq;
  A.kind_curl = vs.kind == SpaceKind::curl;
  A.stride = vs.degree + 1;
  A.n = P.n;
  for (int c = 0; c < 2; ++c) {
    A.px[c] = comp[c]->sx.degree;
    A.py[c] = comp[c]->sy.degree;
    A.nbx[c] = static_cast<int>(comp[c]->nx());
    A.nby[c] = static_cast<int>(comp[c]->ny());
  }
  A.base[0] = 0;
  A.base[1] = vs.Nx();
  A.locsz0 = (A.px[0] + 1) * (A.py[0] + 1);
  A.nloc = A.locsz0 + (A.px[1] + 1) * (A.py[1] + 1);
  A.ntri = A.nloc * (A.nloc + 1) / 2;

  // One upload of every small table (int32 part, then doubles).
  std::vector<int32_t> ih;
  std::vector<int64_t> ioff;
  auto put_i = [&](const int32_t* p, size_t k) {
    ioff.push_back(static_cast<int64_t>(ih.size()));
    ih.insert(ih.end(), p, p + k);
    while (ih.size() % 4) ih.push_back(0);  // 16-byte alignment for int4 loads
  };
  std::vector<int32_t> f2f(full_to_free.begin(), full_to_free.end());
  std::vector<int32_t> fr(P.free_to_full.begin(), P.free_to_full.end());
  put_i(f2f.data(), f2f.size());                // 0
  put_i(fr.data(), fr.size());                  // 1
  put_i(P.box.data(), P.box.size());            // 2
  for (int c = 0; c < 2; ++c)
    for (int d = 0; d < 2; ++d) {
      const Univariate& u = d ? comp[c]->sy : comp[c]->sx;
      std::vector<int32_t> first(ne);
      for (int e = 0; e < ne; ++e) first[e] = u.first_basis(e);
      put_i(first.data(), first.size());
      put_i(u.sup_first.data(), u.sup_first.size());
      put_i(u.sup_last.data(), u.sup_last.size());
    }                                           // 3 + 3*(2c+d) + {0,1,2}
  std::vector<int32_t> pairs;
  pairs.reserve(A.ntri);
  for (int r = 0; r < A.nloc; ++r)
    for (int s = r; s < A.nloc; ++s) pairs.push_back(r | (s << 16));
  put_i(pairs.data(), pairs.size());            // 15
  std::vector<double> dh;
  std::vector<int64_t> doff;
  auto put_d = [&](const std::vector<double>& v) {
    doff.push_back(static_cast<int64_t>(dh.size()));
    dh.insert(dh.end(), v.begin(), v.end());
  };
  for (int c = 0; c < 2; ++c)
    for (int d = 0; d < 2; ++d) {
      put_d(tab[c][d].val);
      put_d(tab[c][d].der);
    }
  put_d(tab[0][0].wq);
  put_d(tab[0][1].wq);

  const double host_prep_ms = std::chrono::duration<double, std::milli>(clk::now() - t_host0).count();
  cudaStream_t st;
  RQB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } guard{st};
  DeviceBuffer d_i, d_d, d_rowptr, d_col, d_el, d_val;
  d_i.alloc(ih.size() * sizeof(int32_t));
  d_i.upload(ih.data(), ih.size() * sizeof(int32_t), st);
  d_d.alloc(dh.size() * sizeof(double));
  d_d.upload(dh.data(), dh.size() * sizeof(double), st);
  const int32_t* ib = d_i.as<int32_t>();
  const double* db = d_d.as<double>();
  A.f2f = ib + ioff[0];
  A.free2full = ib + ioff[1];
  A.box = ib + ioff[2];
  for (int c = 0; c < 2; ++c)
    for (int d = 0; d < 2; ++d) {
      const int k = 3 + 3 * (2 * c + d);
      A.first[c][d] = ib + ioff[k];
      A.supf[c][d] = ib + ioff[k + 1];
      A.supl[c][d] = ib + ioff[k + 2];
      A.val[c][d] = db + doff[2 * (2 * c + d)];
      A.der[c][d] = db + doff[2 * (2 * c + d) + 1];
    }
  A.pairs = ib + ioff[15];
  A.w[0] = db + doff[8];
  A.w[1] = db + doff[9];

  cudaEvent_t ev[4];
  for (auto& x : ev) RQB_CUDA(cudaEventCreate(&x));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]);
    }
  } eg{ev};

  // 1. pattern
  d_rowptr.alloc((P.n + 1) * sizeof(int64_t));
  int64_t* rowptr = d_rowptr.as<int64_t>();
  size_t scan_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, rowptr + 1, rowptr + 1, P.n, st);
  DeviceBuffer d_scan;
  d_scan.alloc(std::max<size_t>(scan_bytes, 16));
  RQB_CUDA(cudaEventRecord(ev[0], st));
  RQB_CUDA(cudaMemsetAsync(rowptr, 0, sizeof(int64_t), st));
  asm_count<<<static_cast<unsigned>((P.n + 255) / 256), 256, 0, st>>>(A, rowptr + 1);
  RQB_CUDA(cudaGetLastError());
  RQB_CUDA(cub::DeviceScan::InclusiveSum(d_scan.p, scan_bytes, rowptr + 1, rowptr + 1, P.n, st));
  int64_t nnz = 0;
  RQB_CUDA(cudaMemcpyAsync(&nnz, rowptr + P.n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  RQB_CUDA(cudaStreamSynchronize(st));
  d_col.alloc(std::max<int64_t>(nnz, 1) * sizeof(int32_t));
  int num_sms = 148;
  {
    int dev = 0;
    RQB_CUDA(cudaGetDevice(&dev));
    RQB_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int64_t warp_blocks = std::min<int64_t>((P.n + 7) / 8, int64_t(num_sms) * 8);
  asm_fill<<<static_cast<unsigned>(warp_blocks), 256, 0, st>>>(A, rowptr, d_col.as<int32_t>());
  RQB_CUDA(cudaGetLastError());
  RQB_CUDA(cudaEventRecord(ev[1], st));

  // 2. element matrices
  const int64_t nel = int64_t(ne) * ne;
  d_el.alloc(2 * nel * A.ntri * sizeof(double));
  A.Kel = d_el.as<double>();
  A.Mel = A.Kel + nel * A.ntri;
  const size_t line = size_t(nq) * A.nloc * 2 * sizeof(double) + nq * sizeof(double);
  const size_t budget = 160 * 1024;
  const int rows = static_cast<int>(std::max<size_t>(1, std::min<size_t>(nq, budget / line)));
  const size_t smem = (size_t((rows * nq + 1) & ~1) + size_t(rows) * nq * A.nloc * 2) * sizeof(double);
  if (smem > 48 * 1024) smem_at_least(asm_element, smem);
  const int threads = A.ntri >= 512 ? 256 : 128;
  asm_element<<<static_cast<unsigned>(nel), threads, smem, st>>>(A, rows);
  RQB_CUDA(cudaGetLastError());
  RQB_CUDA(cudaEventRecord(ev[2], st));

  // 3. colour-ordered gather into the shared pattern
  d_val.alloc(3 * std::max<int64_t>(nnz, 1) * sizeof(double));
  double* K = d_val.as<double>();
  double* C = K + nnz;
  double* M = C + nnz;
  asm_gather<<<static_cast<unsigned>(warp_blocks), 256, 0, st>>>(A, rowptr, d_col.as<int32_t>(), alpha,
                                                                 beta, K, C, M);
  RQB_CUDA(cudaGetLastError());
  RQB_CUDA(cudaEventRecord(ev[3], st));

  RQB_CUDA(cudaStreamSynchronize(st));
  const auto t_d2h0 = clk::now();
  P.rowptr.resize(P.n + 1);
  P.col.resize(nnz);
  RQB_CUDA(cudaMemcpyAsync(P.rowptr.data(), rowptr, (P.n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  RQB_CUDA(cudaMemcpyAsync(P.col.data(), d_col.p, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  if (!keep) {
    P.K.resize(nnz);
    P.C.resize(nnz);
    P.M.resize(nnz);
    RQB_CUDA(cudaMemcpyAsync(P.K.data(), K, nnz * sizeof(double), cudaMemcpyDeviceToHost, st));
    RQB_CUDA(cudaMemcpyAsync(P.C.data(), C, nnz * sizeof(double), cudaMemcpyDeviceToHost, st));
    RQB_CUDA(cudaMemcpyAsync(P.M.data(), M, nnz * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  RQB_CUDA(cudaStreamSynchronize(st));
  if (keep) {
    keep->n = P.n;
    keep->nnz = nnz;
    RQB_CUDA(cudaGetDevice(&keep->device));
    std::swap(keep->d_rowptr.p, d_rowptr.p);
    std::swap(keep->d_rowptr.bytes, d_rowptr.bytes);
    std::swap(keep->d_col.p, d_col.p);
    std::swap(keep->d_col.bytes, d_col.bytes);
    std::swap(keep->d_val.p, d_val.p);
    std::swap(keep->d_val.bytes, d_val.bytes);
  }
  if (ms) {
    float t = 0;
    for (int i = 0; i < 3; ++i) {
      RQB_CUDA(cudaEventElapsedTime(&t, ev[i], ev[i + 1]));
      ms[i] = t;
    }
    ms[3] = host_prep_ms;
    ms[4] = std::chrono::duration<double, std::milli>(clk::now() - t_d2h0).count();
  }
  return P;
}

}  // namespace rqb
