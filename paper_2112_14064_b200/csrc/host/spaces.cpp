// SPDX-License-Identifier: Apache-2.0
// Spline spaces and BASELINE pencil assembly (host input construction).
//
// Restates, in this build's own code, the bookkeeping of the reference
// splines/spaces modules:
//   - open uniform knots with interior multiplicities  (splines.cpp:72-92)
//   - element spans + basis support element ranges      (splines.cpp:25-62)
//   - rIGA separator multiplicities                      (splines.cpp:94-116)
//   - recursive-bisection separator breakpoints          (spaces.cpp:12-24)
//   - curl/div component degree layout                   (spaces.cpp:54-64)
//   - boundary masks em/acoustic                         (spaces.cpp:79-113)
// and the BASELINE forms (BASELINE.json configs; SPEC.md:216-224, 261-264 for
// the quadrature and elimination rules):
//   K = int (div u div v | curl u curl v) + u.v,  M = int u.v,
//   C = alpha M + beta K, (p+1)^2 Gauss points per element, constrained DOFs
//   eliminated, K/C/M on one shared pattern (all support-overlapping pairs).
#include <algorithm>
#include <cmath>
#include <thread>

#include "common.hpp"

namespace rqb {

Univariate make_univariate(int degree, int elems, const std::vector<int>& mult) {
  if (degree < 1) fail(errc::domain, "degree must be at least 1");
  if (elems < 1) fail(errc::domain, "element count must be at least 1");
  if (static_cast<int>(mult.size()) != elems - 1)
    fail(errc::domain, "need one multiplicity per interior breakpoint");
  Univariate u;
  u.degree = degree;
  u.elems = elems;
  u.mult = mult;
  u.knots.assign(degree + 1, 0.0);
  for (int b = 1; b < elems; ++b) {
    const int m = mult[b - 1];
    if (m < 1 || m > degree) fail(errc::domain, "interior multiplicity outside [1, degree]");
    for (int r = 0; r < m; ++r) u.knots.push_back(static_cast<double>(b) / elems);
  }
  for (int r = 0; r <= degree; ++r) u.knots.push_back(1.0);
  u.elem_span.resize(elems);
  int s = degree;
  for (int e = 0; e < elems; ++e) {
    u.elem_span[e] = s;
    if (e < elems - 1) s += mult[e];
  }
  const int nb = u.nbasis();
  u.sup_first.assign(nb, -1);
  u.sup_last.assign(nb, -1);
  for (int e = 0; e < elems; ++e)
    for (int i = u.first_basis(e); i <= u.elem_span[e]; ++i) {
      if (u.sup_first[i] < 0) u.sup_first[i] = e;
      u.sup_last[i] = e;
    }
  return u;
}

namespace {

std::vector<int> bisection_cuts(int elems, int levels) {
  std::vector<int> cuts;
  for (int l = 1; l <= levels; ++l) {
    const int blocks = 1 << l, step = elems / blocks;
    for (int b = 1; b < blocks; b += 2) cuts.push_back(b * step - 1);
  }
  std::sort(cuts.begin(), cuts.end());
  return cuts;
}

// Separator breakpoints get continuity `target` (multiplicity degree-target)
// unless already lower.
Univariate direction(int degree, int elems, const std::vector<int>& seps, int target) {
  std::vector<int> mult(elems - 1, 1);
  for (int b : seps) mult[b] = std::max(mult[b], degree - target);
  return make_univariate(degree, elems, mult);
}

}  // namespace

VectorSpace build_space(SpaceKind kind, int degree, int elems, int levels) {
  if (degree < 2) fail(errc::domain, "vector-valued spaces need degree >= 2");
  if (elems < 2) fail(errc::domain, "need at least 2 elements per direction");
  if (levels < 0) fail(errc::domain, "negative partition level");
  if (levels > 0) {
    if (levels > 30 || elems % (1 << levels) != 0)
      fail(errc::domain, "element count not divisible by 2^levels");
    if (elems / (1 << levels) < 2) fail(errc::domain, "macroelements must span >= 2 elements");
  }
  VectorSpace vs;
  vs.kind = kind;
  vs.degree = degree;
  vs.elems = elems;
  vs.levels = levels;
  vs.separators = bisection_cuts(elems, levels);
  const Univariate hi = direction(degree, elems, vs.separators, 1);
  const Univariate lo = direction(degree - 1, elems, vs.separators, 0);
  if (kind == SpaceKind::curl) {
    vs.cx = Tensor2{lo, hi};
    vs.cy = Tensor2{hi, lo};
  } else {
    vs.cx = Tensor2{hi, lo};
    vs.cy = Tensor2{lo, hi};
  }
  return vs;
}

std::vector<int64_t> boundary_mask(const VectorSpace& vs) {
  std::vector<int64_t> mask;
  const int64_t nx1 = vs.cx.nx(), ny1 = vs.cx.ny(), nx2 = vs.cy.nx(), ny2 = vs.cy.ny();
  const int64_t Nx = vs.Nx();
  if (vs.kind == SpaceKind::curl) {
    // E x n = 0: x-component on horizontal edges, y-component on vertical ones.
    for (int64_t i = 0; i < nx1; ++i) {
      mask.push_back(i);
      mask.push_back((ny1 - 1) * nx1 + i);
    }
    for (int64_t j = 0; j < ny2; ++j) {
      mask.push_back(Nx + j * nx2);
      mask.push_back(Nx + j * nx2 + nx2 - 1);
    }
  } else {
    // u . n = 0 on all four (rigid) edges.
    for (int64_t j = 0; j < ny1; ++j) {
      mask.push_back(j * nx1);
      mask.push_back(j * nx1 + nx1 - 1);
    }
    for (int64_t i = 0; i < nx2; ++i) {
      mask.push_back(Nx + i);
      mask.push_back(Nx + (ny2 - 1) * nx2 + i);
    }
  }
  std::sort(mask.begin(), mask.end());
  mask.erase(std::unique(mask.begin(), mask.end()), mask.end());
  return mask;
}

namespace {

constexpr int kMaxP = kMaxAsmDegree;

// Gauss-Legendre nodes/weights on [-1,1] (Newton on P_n).
void gauss_legendre(int n, double* x, double* w) {
  for (int i = 0; i < n; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= n; ++k) {
        const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    double p0 = 1.0, p1 = z;
    for (int k = 2; k <= n; ++k) {
      const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    dp = n * (z * p1 - p0) / (z * z - 1.0);
    x[n - 1 - i] = z;
    w[n - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}

// Degree-p B-spline values and first derivatives of the p+1 bases s-p..s at
// u, from the Cox-de Boor definition (0/0 := 0).
void basis_eval(const std::vector<double>& U, int p, int s, double u, double* val, double* der) {
  double N[kMaxP + 2], Nn[kMaxP + 2], Np[kMaxP + 2];
  N[0] = 1.0;
  Np[0] = 1.0;
  for (int k = 1; k <= p; ++k) {
    if (k == p)
      for (int r = 0; r < p; ++r) Np[r] = N[r];
    for (int r = 0; r <= k; ++r) {
      const int i = s - k + r;
      double v = 0.0;
      if (r >= 1) {
        const double den = U[i + k] - U[i];
        if (den > 0) v += (u - U[i]) / den * N[r - 1];
      }
      if (r <= k - 1) {
        const double den = U[i + k + 1] - U[i + 1];
        if (den > 0) v += (U[i + k + 1] - u) / den * N[r];
      }
      Nn[r] = v;
    }
    for (int r = 0; r <= k; ++r) N[r] = Nn[r];
  }
  for (int r = 0; r <= p; ++r) {
    val[r] = N[r];
    if (p == 0) {
      der[r] = 0.0;
      continue;
    }
    const int i = s - p + r;
    double d = 0.0;
    if (r >= 1) {
      const double den = U[i + p] - U[i];
      if (den > 0) d += p / den * Np[r - 1];
    }
    if (r <= p - 1) {
      const double den = U[i + p + 1] - U[i + 1];
      if (den > 0) d -= p / den * Np[r];
    }
    der[r] = d;
  }
}

// First basis index whose support reaches element lo / last reaching hi.
void overlap_range(const Univariate& u, int lo, int hi, int* first, int* last) {
  const int nb = u.nbasis();
  int a = 0;
  while (a < nb && u.sup_last[a] < lo) ++a;
  int b = nb - 1;
  while (b >= 0 && u.sup_first[b] > hi) --b;
  *first = a;
  *last = b;
}

}  // namespace

void QuadTable::build(const Univariate& u, const double* gx, const double* gw, int nq_) {
  p = u.degree;
  nq = nq_;
  const int ne = u.elems;
  val.assign(static_cast<size_t>(ne) * nq * (p + 1), 0.0);
  der.assign(val.size(), 0.0);
  wq.assign(static_cast<size_t>(ne) * nq, 0.0);
  for (int e = 0; e < ne; ++e) {
    const double x0 = static_cast<double>(e) / ne, x1 = static_cast<double>(e + 1) / ne;
    const double h = x1 - x0;
    for (int q = 0; q < nq; ++q) {
      const double x = x0 + 0.5 * (gx[q] + 1.0) * h;
      const size_t o = (static_cast<size_t>(e) * nq + q) * (p + 1);
      basis_eval(u.knots, p, u.elem_span[e], x, &val[o], &der[o]);
      wq[static_cast<size_t>(e) * nq + q] = 0.5 * h * gw[q];
    }
  }
}

void quad_tables(const VectorSpace& vs, QuadTable tab[2][2]) {
  if (vs.degree > kMaxP) fail(errc::domain, "degree too large for assembly tables");
  const int nq = vs.degree + 1;
  double gx[kMaxP + 1], gw[kMaxP + 1];
  gauss_legendre(nq, gx, gw);
  const Tensor2* comp[2] = {&vs.cx, &vs.cy};
  for (int c = 0; c < 2; ++c) {
    tab[c][0].build(comp[c]->sx, gx, gw, nq);
    tab[c][1].build(comp[c]->sy, gx, gw, nq);
  }
}

void free_numbering(const VectorSpace& vs, std::vector<int64_t>* full_to_free,
                    std::vector<int64_t>* free_to_full, const std::vector<int64_t>* mask_in) {
  const std::vector<int64_t> mask = mask_in ? *mask_in : boundary_mask(vs);
  const int64_t N = vs.N();
  full_to_free->assign(N, -1);
  free_to_full->clear();
  free_to_full->reserve(N - mask.size());
  size_t mi = 0;
  for (int64_t g = 0; g < N; ++g) {
    if (mi < mask.size() && mask[mi] == g) {
      ++mi;
      continue;
    }
    (*full_to_free)[g] = static_cast<int64_t>(free_to_full->size());
    free_to_full->push_back(g);
  }
}

std::vector<int32_t> support_boxes(const VectorSpace& vs, const std::vector<int64_t>& free_to_full) {
  const Tensor2* comp[2] = {&vs.cx, &vs.cy};
  const int64_t base[2] = {0, vs.Nx()};
  const int64_t n = static_cast<int64_t>(free_to_full.size());
  std::vector<int32_t> box(4 * n);
  for (int64_t k = 0; k < n; ++k) {
    const int64_t g = free_to_full[k];
    const int c = g >= vs.Nx() ? 1 : 0;
    const int64_t l = g - base[c];
    const int i = static_cast<int>(l % comp[c]->nx()), j = static_cast<int>(l / comp[c]->nx());
    box[4 * k + 0] = comp[c]->sx.sup_first[i];
    box[4 * k + 1] = comp[c]->sx.sup_last[i];
    box[4 * k + 2] = comp[c]->sy.sup_first[j];
    box[4 * k + 3] = comp[c]->sy.sup_last[j];
  }
  return box;
}

Pencil assemble_pencil(const VectorSpace& vs, double alpha, double beta, const std::vector<int64_t>* mask,
                       std::vector<int64_t>* full_to_free_out) {
  if (vs.degree > kMaxP) fail(errc::domain, "degree too large for assembly tables");
  Pencil P;
  P.elems = vs.elems;
  P.n_full = vs.N();
  std::vector<int64_t> full_to_free;
  free_numbering(vs, &full_to_free, &P.free_to_full, mask);
  P.n = static_cast<int64_t>(P.free_to_full.size());
  const Tensor2* comp[2] = {&vs.cx, &vs.cy};
  const int64_t base[2] = {0, vs.Nx()};

  // Support boxes and shared pattern (all support-overlapping free pairs).
  P.box = support_boxes(vs, P.free_to_full);
  P.rowptr.assign(P.n + 1, 0);
  auto row_cols = [&](int64_t k, std::vector<int32_t>& out) {
    out.clear();
    const int32_t* b = &P.box[4 * k];
    for (int c = 0; c < 2; ++c) {
      int i0, i1, j0, j1;
      overlap_range(comp[c]->sx, b[0], b[1], &i0, &i1);
      overlap_range(comp[c]->sy, b[2], b[3], &j0, &j1);
      for (int j = j0; j <= j1; ++j)
        for (int i = i0; i <= i1; ++i) {
          const int64_t f = full_to_free[base[c] + static_cast<int64_t>(j) * comp[c]->nx() + i];
          if (f >= 0) out.push_back(static_cast<int32_t>(f));
        }
    }
  };
  {
    std::vector<int32_t> tmp;
    for (int64_t k = 0; k < P.n; ++k) {
      row_cols(k, tmp);
      P.rowptr[k + 1] = P.rowptr[k] + static_cast<int64_t>(tmp.size());
    }
    P.col.resize(P.rowptr[P.n]);
    const unsigned nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nth; ++t)
      th.emplace_back([&, t] {
        std::vector<int32_t> loc;
        for (int64_t k = t; k < P.n; k += nth) {
          row_cols(k, loc);
          std::copy(loc.begin(), loc.end(), P.col.begin() + P.rowptr[k]);
        }
      });
    for (auto& x : th) x.join();
  }
  const int64_t nnz = P.rowptr[P.n];
  P.K.assign(nnz, 0.0);
  P.M.assign(nnz, 0.0);

  // Quadrature tables.
  const int nq = vs.degree + 1;
  QuadTable tab[2][2];  // [component][direction]
  quad_tables(vs, tab);
  const bool curl = vs.kind == SpaceKind::curl;
  const int ne = vs.elems;

  // Element rows of one colour (stride p+1 in y) share no DOF, so each colour
  // phase is race-free and the summation order is thread-count independent.
  auto do_row = [&](int ey, std::vector<double>& Kl, std::vector<double>& Ml,
                    std::vector<int64_t>& dof, std::vector<double>& vals) {
    for (int ex = 0; ex < ne; ++ex) {
      // Local DOFs: component 0 then 1, (a,b) with a fastest.
      int nloc = 0;
      int locsz[2];
      for (int c = 0; c < 2; ++c) {
        const int px = comp[c]->sx.degree, py = comp[c]->sy.degree;
        const int fx = comp[c]->sx.first_basis(ex), fy = comp[c]->sy.first_basis(ey);
        for (int b = 0; b <= py; ++b)
          for (int a = 0; a <= px; ++a)
            dof[nloc++] = full_to_free[base[c] + static_cast<int64_t>(fy + b) * comp[c]->nx() + fx + a];
        locsz[c] = (px + 1) * (py + 1);
      }
      std::fill(Kl.begin(), Kl.begin() + nloc * nloc, 0.0);
      std::fill(Ml.begin(), Ml.begin() + nloc * nloc, 0.0);
      // vals layout per local dof: value (component), curl/div
      for (int qy = 0; qy < nq; ++qy)
        for (int qx = 0; qx < nq; ++qx) {
          const double w = tab[0][0].w(ex, qx) * tab[0][1].w(ey, qy);
          int o = 0;
          for (int c = 0; c < 2; ++c) {
            const QuadTable& TX = tab[c][0];
            const QuadTable& TY = tab[c][1];
            const double* vx = TX.v(ex, qx);
            const double* dx = TX.d(ex, qx);
            const double* vy = TY.v(ey, qy);
            const double* dy = TY.d(ey, qy);
            for (int b = 0; b <= TY.p; ++b)
              for (int a = 0; a <= TX.p; ++a, ++o) {
                const double val = vx[a] * vy[b];
                double dd;
                if (!curl)
                  dd = c == 0 ? dx[a] * vy[b] : vx[a] * dy[b];  // div
                else
                  dd = c == 0 ? -vx[a] * dy[b] : dx[a] * vy[b];  // curl
                vals[2 * o] = val;
                vals[2 * o + 1] = dd;
              }
          }
          for (int r = 0; r < nloc; ++r) {
            const int cr = r < locsz[0] ? 0 : 1;
            const double vr = w * vals[2 * r], dr = w * vals[2 * r + 1];
            for (int s = r; s < nloc; ++s) {
              const int cs = s < locsz[0] ? 0 : 1;
              const double mm = cr == cs ? vr * vals[2 * s] : 0.0;
              Kl[r * nloc + s] += dr * vals[2 * s + 1] + mm;
              Ml[r * nloc + s] += mm;
            }
          }
        }
      // exact symmetry: mirror the upper triangle
      for (int r = 0; r < nloc; ++r)
        for (int s = 0; s < r; ++s) {
          Kl[r * nloc + s] = Kl[s * nloc + r];
          Ml[r * nloc + s] = Ml[s * nloc + r];
        }
      for (int r = 0; r < nloc; ++r) {
        const int64_t fr = dof[r];
        if (fr < 0) continue;
        const int32_t* cb = P.col.data() + P.rowptr[fr];
        const int32_t* ce = P.col.data() + P.rowptr[fr + 1];
        for (int s = 0; s < nloc; ++s) {
          const int64_t fs = dof[s];
          if (fs < 0) continue;
          const int32_t* it = std::lower_bound(cb, ce, static_cast<int32_t>(fs));
          if (it == ce || *it != fs) fail(errc::assembly, "pattern misses an element pair");
          const int64_t pos = it - P.col.data();
          P.K[pos] += Kl[r * nloc + s];
          P.M[pos] += Ml[r * nloc + s];
        }
      }
    }
  };
  const int stride = vs.degree + 1;
  const unsigned nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  for (int colour = 0; colour < stride; ++colour) {
    std::vector<int> rows;
    for (int ey = colour; ey < ne; ey += stride) rows.push_back(ey);
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nth; ++t)
      th.emplace_back([&, t] {
        const int maxloc = 2 * (vs.degree + 1) * vs.degree;
        std::vector<double> Kl(maxloc * maxloc), Ml(maxloc * maxloc), vals(2 * maxloc);
        std::vector<int64_t> dof(maxloc);
        for (size_t r = t; r < rows.size(); r += nth) do_row(rows[r], Kl, Ml, dof, vals);
      });
    for (auto& x : th) x.join();
  }
  P.C.resize(nnz);
  for (int64_t k = 0; k < nnz; ++k) P.C[k] = alpha * P.M[k] + beta * P.K[k];
  if (full_to_free_out) *full_to_free_out = std::move(full_to_free);
  return P;
}

// The paper's vibroacoustic pencil (SPEC.md:225-232,
// assemble_acoustic): u . n = 0 on the rigid edges only (the absorbing ones
// stay free), K = int rho c^2 div u div v + int_{Gamma_A} alpha (u.n)(v.n),
// C = int_{Gamma_A} beta (u.n)(v.n), M = int rho u.v, all real. On an edge
// only the normal component's bases of the last (or first) index across the
// edge are nonzero (open knot vectors: value 1 there), so the edge integral is
// the 1-D mass matrix of the tangential univariate space, integrated with p+1
// Gauss points per element.
Pencil assemble_acoustic(const VectorSpace& vs, double rho, double c, double alpha, double beta, int absorbing) {
  if (vs.kind != SpaceKind::div) fail(errc::domain, "the acoustic problem lives in H(div)");
  if (!(rho > 0 && c > 0 && alpha > 0 && beta > 0)) fail(errc::domain, "acoustic material: rho, c, alpha, beta > 0");
  if (absorbing < 0 || absorbing > 15) fail(errc::domain, "absorbing edges: bit mask of left 1, right 2, bottom 4, top 8");
  // rigid edges: the normal component's boundary DOFs
  std::vector<int64_t> mask;
  const int64_t nx1 = vs.cx.nx(), ny1 = vs.cx.ny(), nx2 = vs.cy.nx(), ny2 = vs.cy.ny(), Nx = vs.Nx();
  for (int64_t j = 0; j < ny1; ++j) {
    if (!(absorbing & 1)) mask.push_back(j * nx1);
    if (!(absorbing & 2)) mask.push_back(j * nx1 + nx1 - 1);
  }
  for (int64_t i = 0; i < nx2; ++i) {
    if (!(absorbing & 4)) mask.push_back(Nx + i);
    if (!(absorbing & 8)) mask.push_back(Nx + (ny2 - 1) * nx2 + i);
  }
  std::sort(mask.begin(), mask.end());
  std::vector<int64_t> full_to_free;
  Pencil P = assemble_pencil(vs, 0.0, 0.0, &mask, &full_to_free);
  const int64_t nnz = P.rowptr[P.n];
  const double rc2 = rho * c * c;
  for (int64_t k = 0; k < nnz; ++k) {
    P.K[k] = rc2 * (P.K[k] - P.M[k]);  // the BASELINE K carries div-div + u.v
    P.M[k] = rho * P.M[k];
    P.C[k] = 0.0;
  }
  auto add = [&](int64_t fr, int64_t fs, double v) {
    const int32_t* cb = P.col.data() + P.rowptr[fr];
    const int32_t* ce = P.col.data() + P.rowptr[fr + 1];
    const int32_t* it = std::lower_bound(cb, ce, static_cast<int32_t>(fs));
    if (it == ce || *it != fs) fail(errc::assembly, "pattern misses an edge pair");
    const int64_t pos = it - P.col.data();
    P.K[pos] += alpha * v;
    P.C[pos] += beta * v;
  };
  const int nq = vs.degree + 1;
  std::vector<double> gx(nq), gw(nq);
  gauss_legendre(nq, gx.data(), gw.data());
  for (int edge = 0; edge < 4; ++edge) {
    if (!(absorbing & (1 << edge))) continue;
    // vertical edges (left/right): x-component, tangential univariate cx.sy;
    // horizontal edges (bottom/top): y-component, tangential cy.sx
    const bool vert = edge < 2;
    const Tensor2& T = vert ? vs.cx : vs.cy;
    const Univariate& tu = vert ? T.sy : T.sx;
    const int64_t nxt = T.nx();
    const int64_t across = (edge == 0 || edge == 2) ? 0 : (vert ? T.nx() - 1 : T.ny() - 1);
    const int64_t base = vert ? 0 : Nx;
    auto dof = [&](int64_t t) {  // full index of the normal-component basis (t along the edge)
      return base + (vert ? t * nxt + across : across * nxt + t);
    };
    const int p = tu.degree;
    std::vector<double> val(p + 1), der(p + 1);
    for (int e = 0; e < tu.elems; ++e) {
      const int span = tu.elem_span[e];
      const double u0 = tu.knots[span], u1 = tu.knots[span + 1], h = u1 - u0;
      for (int q = 0; q < nq; ++q) {
        const double u = u0 + 0.5 * (gx[q] + 1.0) * h, w = 0.5 * h * gw[q];
        basis_eval(tu.knots, p, span, u, val.data(), der.data());
        for (int a = 0; a <= p; ++a) {
          const int64_t fa = full_to_free[dof(span - p + a)];
          if (fa < 0) continue;
          for (int b = 0; b <= p; ++b) {
            const int64_t fb = full_to_free[dof(span - p + b)];
            if (fb < 0) continue;
            add(fa, fb, w * val[a] * val[b]);
          }
        }
      }
    }
  }
  return P;
}


// The paper's conductive electromagnetic pencil (§2.1; SPEC.md:216-224,
// assemble_em): H(curl) space with E x n = 0, K = int curl u (-1/mu) curl v,
// M = int eps u.v, C = int u . (-i sigma) v with sigma = diag(sigma_x(y),
// sigma_y(y)) piecewise constant over horizontal layers; returned as real K, M
// and the real D with C = -i D (the pencil is complex through C only).
Pencil assemble_em(const VectorSpace& vs, double mu, double eps, const std::vector<EmLayer>& layers,
                   std::vector<double>* D_out) {
  if (vs.kind != SpaceKind::curl) fail(errc::domain, "the electromagnetic problem lives in H(curl)");
  if (!(mu > 0 && eps > 0)) fail(errc::domain, "mu and eps must be positive");
  for (const EmLayer& L : layers)
    if (!(L.y1 > L.y0) || L.sx < 0 || L.sy < 0) fail(errc::domain, "layers: y0 < y1, sigma >= 0");
  std::vector<int64_t> full_to_free;
  Pencil P = assemble_pencil(vs, 0.0, 0.0, nullptr, &full_to_free);
  const int64_t nnz = P.rowptr[P.n];
  for (int64_t k = 0; k < nnz; ++k) {
    P.K[k] = -(P.K[k] - P.M[k]) / mu;  // the BASELINE K carries curl-curl + u.v
    P.M[k] = eps * P.M[k];
    P.C[k] = 0.0;
  }
  std::vector<double>& D = *D_out;
  D.assign(nnz, 0.0);
  const int nq = vs.degree + 1, ne = vs.elems;
  QuadTable tab[2][2];
  quad_tables(vs, tab);
  double gx[kMaxP + 1], gw[kMaxP + 1];
  gauss_legendre(nq, gx, gw);
  const Tensor2* comp[2] = {&vs.cx, &vs.cy};
  const int64_t base[2] = {0, vs.Nx()};
  auto sigma_at = [&](double y, int c) {
    for (const EmLayer& L : layers)
      if (y >= L.y0 && y < L.y1) return c == 0 ? L.sx : L.sy;
    return 0.0;
  };
  std::vector<int64_t> dof;
  std::vector<double> vals;
  for (int ey = 0; ey < ne; ++ey)
    for (int ex = 0; ex < ne; ++ex)
      for (int c = 0; c < 2; ++c) {
        const QuadTable& TX = tab[c][0];
        const QuadTable& TY = tab[c][1];
        const int fx = comp[c]->sx.first_basis(ex), fy = comp[c]->sy.first_basis(ey);
        dof.clear();
        for (int b = 0; b <= TY.p; ++b)
          for (int a = 0; a <= TX.p; ++a)
            dof.push_back(full_to_free[base[c] + static_cast<int64_t>(fy + b) * comp[c]->nx() + fx + a]);
        const int nl = static_cast<int>(dof.size());
        for (int qy = 0; qy < nq; ++qy) {
          const double y = (ey + 0.5 * (gx[qy] + 1.0)) / ne;
          const double sg = sigma_at(y, c);
          if (sg == 0.0) continue;
          for (int qx = 0; qx < nq; ++qx) {
            const double w = TX.w(ex, qx) * TY.w(ey, qy) * sg;
            vals.assign(nl, 0.0);
            const double* vx = TX.v(ex, qx);
            const double* vy = TY.v(ey, qy);
            for (int b = 0, o = 0; b <= TY.p; ++b)
              for (int a = 0; a <= TX.p; ++a, ++o) vals[o] = vx[a] * vy[b];
            for (int r = 0; r < nl; ++r) {
              if (dof[r] < 0) continue;
              const int32_t* cb = P.col.data() + P.rowptr[dof[r]];
              const int32_t* ce = P.col.data() + P.rowptr[dof[r] + 1];
              for (int q = 0; q < nl; ++q) {
                if (dof[q] < 0) continue;
                const int32_t* it = std::lower_bound(cb, ce, static_cast<int32_t>(dof[q]));
                if (it == ce || *it != dof[q]) fail(errc::assembly, "pattern misses an element pair");
                D[it - P.col.data()] += w * vals[r] * vals[q];
              }
            }
          }
        }
      }
  return P;
}

}  // namespace rqb
