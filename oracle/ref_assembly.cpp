// SPDX-License-Identifier: Apache-2.0
// ORACLE — TEST INFRASTRUCTURE ONLY. Independent BASELINE pencil assembly on
// the reference's own substrate (compiled into oracle/_ref/liboracle_ref.so
// from /root/reference/proj): spaces from build_iga_space / build_riga_space
// (spaces.cpp:33-77), constrained DOFs from boundary_mask (spaces.cpp:79-113),
// basis values and first derivatives from eval_basis_derivatives
// (splines.cpp:143-207), physical values / curl / div through piola_map
// (spaces.cpp:115-132). The element loop, the Gauss rule and the CSR build are
// written here independently of the product's assembler
// (paper_2112_14064_b200/csrc/host/spaces.cpp, csrc/cuda/assembly.cu), so the
// product's K, C, M are pinned against a second route and the reference CPU
// arm (bench.py --impl reference) gets its pencil without loading the product.
//
// BASELINE.json configs: K_ij = int (div phi_i div phi_j | curl phi_i curl phi_j)
// + phi_i . phi_j, M_ij = int phi_i . phi_j, C = alpha M + beta K, (p+1)^2
// Gauss points per element, constrained DOFs eliminated (H(div): zero normal
// trace, boundary_mask(acoustic, all edges); H(curl): zero tangential trace,
// boundary_mask(em)).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "rigaqep/spaces.hpp"
#include "rigaqep/splines.hpp"

namespace {

thread_local std::string g_err;

// Gauss-Legendre nodes/weights on [-1, 1] by Newton iteration on P_n.
void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < n; ++i) {
    double z = std::cos(pi * (i + 0.75) / (n + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= n; ++k) {
        const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (n == 1) p1 = z, p0 = 1.0;
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    x[n - 1 - i] = z;
    w[n - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}

struct DirTable {  // per element e of one direction: values / derivatives at the Gauss points
  int p = 0, nq = 0;
  std::vector<double> val, der;  // [e][q][j], j = 0..p
  std::vector<double> wq;        // [e][q] physical-parameter weight (element length * w / 2)
  std::vector<int> base;         // first basis on element e
};

DirTable tabulate(const rq::UnivariateSpace& s, const std::vector<double>& gx, const std::vector<double>& gw) {
  DirTable t;
  t.p = s.degree();
  t.nq = static_cast<int>(gx.size());
  const int ne = s.elem_count(), p1 = t.p + 1;
  t.val.resize(static_cast<size_t>(ne) * t.nq * p1);
  t.der.resize(t.val.size());
  t.wq.resize(static_cast<size_t>(ne) * t.nq);
  t.base.resize(ne);
  for (int e = 0; e < ne; ++e) {
    const double a = s.elem_x0(e), b = s.elem_x1(e);
    t.base[e] = s.span_base(e);
    for (int q = 0; q < t.nq; ++q) {
      const double u = a + 0.5 * (gx[q] + 1.0) * (b - a);
      t.wq[static_cast<size_t>(e) * t.nq + q] = 0.5 * (b - a) * gw[q];
      const rq::BasisDerivEval d = rq::eval_basis_derivatives(s.kv(), u, 1);
      if (d.span - t.p != t.base[e]) throw rq::Error(rq::errc::assembly, "span/base mismatch");
      for (int j = 0; j < p1; ++j) {
        t.val[(static_cast<size_t>(e) * t.nq + q) * p1 + j] = d.value(0, j);
        t.der[(static_cast<size_t>(e) * t.nq + q) * p1 + j] = d.value(1, j);
      }
    }
  }
  return t;
}

struct RefPencil {
  int64_t n_full = 0, n = 0;
  std::vector<int64_t> rowptr;
  std::vector<int32_t> col;
  std::vector<double> K, C, M;
  std::vector<int32_t> box;  // per free DOF {x0, x1, y0, y1}
};

RefPencil assemble(int kind, int p, int ne, int levels, double alpha, double beta) {
  const rq::SpaceKind k = kind == 0 ? rq::SpaceKind::curl : rq::SpaceKind::divergence;
  const rq::BoxGeometry geom{};
  const rq::VectorSpace vs =
      levels > 0 ? rq::build_riga_space(k, p, ne, levels, geom) : rq::build_iga_space(k, p, ne, geom);
  const std::vector<long> mask =
      rq::boundary_mask(vs, kind == 0 ? rq::ModelProblem::em : rq::ModelProblem::acoustic);
  RefPencil R;
  R.n_full = vs.N();
  std::vector<int32_t> free_id(R.n_full, 0);
  for (long c : mask) free_id[c] = -1;
  int64_t nfree = 0;
  for (int64_t g = 0; g < R.n_full; ++g)
    if (free_id[g] >= 0) free_id[g] = static_cast<int32_t>(nfree++);
  R.n = nfree;
  const rq::TensorSpace2D* comp[2] = {&vs.comp_x, &vs.comp_y};
  R.box.resize(4 * nfree);
  {
    int64_t g = 0;
    for (int c = 0; c < 2; ++c)
      for (int j = 0; j < comp[c]->ny(); ++j)
        for (int i = 0; i < comp[c]->nx(); ++i, ++g) {
          const int32_t f = free_id[g];
          if (f < 0) continue;
          R.box[4 * f + 0] = comp[c]->sx.support_first_elem(i);
          R.box[4 * f + 1] = comp[c]->sx.support_last_elem(i);
          R.box[4 * f + 2] = comp[c]->sy.support_first_elem(j);
          R.box[4 * f + 3] = comp[c]->sy.support_last_elem(j);
        }
  }
  std::vector<double> gx, gw;
  gauss_legendre(p + 1, gx, gw);
  // per component: x- and y-direction tables
  DirTable tx[2] = {tabulate(comp[0]->sx, gx, gw), tabulate(comp[1]->sx, gx, gw)};
  DirTable ty[2] = {tabulate(comp[0]->sy, gx, gw), tabulate(comp[1]->sy, gx, gw)};
  const int nq = p + 1;
  const double detj = rq::piola_factors(k, geom).detj;  // physical measure of the parametric element
  // local DOFs of an element: component c, local (a, b) -> global
  auto local_dofs = [&](int ex, int ey, std::vector<int32_t>& ids, std::vector<int>& cc, std::vector<int>& la,
                        std::vector<int>& lb) {
    ids.clear(), cc.clear(), la.clear(), lb.clear();
    int64_t off = 0;
    for (int c = 0; c < 2; ++c) {
      const int px = tx[c].p, py = ty[c].p;
      for (int b = 0; b <= py; ++b)
        for (int a = 0; a <= px; ++a) {
          const int i = tx[c].base[ex] + a, j = ty[c].base[ey] + b;
          const int32_t f = free_id[off + comp[c]->index(i, j)];
          if (f < 0) continue;
          ids.push_back(f), cc.push_back(c), la.push_back(a), lb.push_back(b);
        }
      off += comp[c]->dofs();
    }
  };
  // pattern: DOF pairs sharing an element
  std::vector<std::vector<int32_t>> rows(nfree);
  std::vector<int32_t> ids;
  std::vector<int> cc, la, lb;
  for (int ey = 0; ey < ne; ++ey)
    for (int ex = 0; ex < ne; ++ex) {
      local_dofs(ex, ey, ids, cc, la, lb);
      for (int32_t r : ids)
        for (int32_t c : ids) rows[r].push_back(c);
    }
  R.rowptr.assign(nfree + 1, 0);
  for (int64_t r = 0; r < nfree; ++r) {
    auto& v = rows[r];
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    R.rowptr[r + 1] = R.rowptr[r] + static_cast<int64_t>(v.size());
  }
  R.col.resize(R.rowptr[nfree]);
  for (int64_t r = 0; r < nfree; ++r) {
    std::copy(rows[r].begin(), rows[r].end(), R.col.begin() + R.rowptr[r]);
    std::vector<int32_t>().swap(rows[r]);
  }
  R.K.assign(R.col.size(), 0.0);
  R.M.assign(R.col.size(), 0.0);
  // element matrices
  std::vector<double> val, dv;  // per local DOF, per Gauss point: value (2), curl/div
  for (int ey = 0; ey < ne; ++ey)
    for (int ex = 0; ex < ne; ++ex) {
      local_dofs(ex, ey, ids, cc, la, lb);
      const int nl = static_cast<int>(ids.size());
      val.assign(static_cast<size_t>(nl) * nq * nq * 2, 0.0);
      dv.assign(static_cast<size_t>(nl) * nq * nq, 0.0);
      std::vector<double> wts(nq * nq);
      for (int qy = 0; qy < nq; ++qy)
        for (int qx = 0; qx < nq; ++qx)
          wts[qy * nq + qx] = detj * tx[0].wq[static_cast<size_t>(ex) * nq + qx] * ty[0].wq[static_cast<size_t>(ey) * nq + qy];
      for (int l = 0; l < nl; ++l) {
        const int c = cc[l];
        const DirTable &X = tx[c], &Y = ty[c];
        const int px1 = X.p + 1, py1 = Y.p + 1;
        for (int qy = 0; qy < nq; ++qy)
          for (int qx = 0; qx < nq; ++qx) {
            const double bx = X.val[(static_cast<size_t>(ex) * nq + qx) * px1 + la[l]];
            const double dbx = X.der[(static_cast<size_t>(ex) * nq + qx) * px1 + la[l]];
            const double by = Y.val[(static_cast<size_t>(ey) * nq + qy) * py1 + lb[l]];
            const double dby = Y.der[(static_cast<size_t>(ey) * nq + qy) * py1 + lb[l]];
            std::array<double, 2> v{0.0, 0.0};
            std::array<double, 4> g{0.0, 0.0, 0.0, 0.0};
            v[c] = bx * by;
            g[2 * c + 0] = dbx * by;  // d/dxi
            g[2 * c + 1] = bx * dby;  // d/deta
            const rq::PiolaApplied pa = rq::piola_map(k, geom, v, g);
            const size_t q = static_cast<size_t>(qy) * nq + qx;
            val[(static_cast<size_t>(l) * nq * nq + q) * 2 + 0] = pa.value[0];
            val[(static_cast<size_t>(l) * nq * nq + q) * 2 + 1] = pa.value[1];
            dv[static_cast<size_t>(l) * nq * nq + q] = pa.curl_or_div;
          }
      }
      for (int a = 0; a < nl; ++a) {
        const int64_t r = ids[a];
        const int32_t* rb = R.col.data() + R.rowptr[r];
        const int64_t rl = R.rowptr[r + 1] - R.rowptr[r];
        for (int b = 0; b < nl; ++b) {
          double m = 0.0, kk = 0.0;
          for (int q = 0; q < nq * nq; ++q) {
            const size_t ia = static_cast<size_t>(a) * nq * nq + q, ib = static_cast<size_t>(b) * nq * nq + q;
            m += wts[q] * (val[2 * ia] * val[2 * ib] + val[2 * ia + 1] * val[2 * ib + 1]);
            kk += wts[q] * dv[ia] * dv[ib];
          }
          const int64_t pos = std::lower_bound(rb, rb + rl, ids[b]) - rb;
          R.M[R.rowptr[r] + pos] += m;
          R.K[R.rowptr[r] + pos] += kk + m;
        }
      }
    }
  R.C.resize(R.K.size());
  for (size_t e = 0; e < R.K.size(); ++e) R.C[e] = alpha * R.M[e] + beta * R.K[e];
  return R;
}

}  // namespace

extern "C" {

const char* ref_assemble_last_error() { return g_err.c_str(); }

// BASELINE pencil on the reference's spaces (kind 0 curl, 1 div; levels =
// rIGA bisection levels, 0 = IGA). Returns an opaque handle.
int ref_assemble(int kind, int degree, int elems, int levels, double alpha, double beta, void** out) {
  try {
    *out = new RefPencil(assemble(kind, degree, elems, levels, alpha, beta));
    return 0;
  } catch (const rq::Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

void ref_assemble_dims(const void* h, int64_t* n_full, int64_t* n, int64_t* nnz) {
  const RefPencil* R = static_cast<const RefPencil*>(h);
  *n_full = R->n_full;
  *n = R->n;
  *nnz = static_cast<int64_t>(R->col.size());
}

// Any output may be NULL.
void ref_assemble_copy(const void* h, int64_t* rowptr, int32_t* col, double* K, double* C, double* M,
                       int32_t* box) {
  const RefPencil* R = static_cast<const RefPencil*>(h);
  if (rowptr) std::memcpy(rowptr, R->rowptr.data(), sizeof(int64_t) * R->rowptr.size());
  if (col) std::memcpy(col, R->col.data(), sizeof(int32_t) * R->col.size());
  if (K) std::memcpy(K, R->K.data(), sizeof(double) * R->K.size());
  if (C) std::memcpy(C, R->C.data(), sizeof(double) * R->C.size());
  if (M) std::memcpy(M, R->M.data(), sizeof(double) * R->M.size());
  if (box) std::memcpy(box, R->box.data(), sizeof(int32_t) * R->box.size());
}

void ref_assemble_destroy(void* h) { delete static_cast<RefPencil*>(h); }

}  // extern "C"
