// SPDX-License-Identifier: Apache-2.0
// ORACLE — TEST INFRASTRUCTURE ONLY. extern "C" shim over the reference's own
// sources (compiled from /root/reference/proj by oracle/Makefile into
// oracle/_ref/): spaces (spaces.cpp:33-113, splines.cpp:25-62) and the kern::
// backend table (kernels.hpp:17-69), so tests can pin the product's spaces
// and the oracle's restated kernels against the reference itself.
#include <cstdint>
#include <cstring>

#include <string>
#include <vector>

#include "rigaqep/kernels.hpp"
#include "rigaqep/spaces.hpp"
#include "rigaqep/sparse.hpp"

extern "C" {

// Full-space sizes + per-DOF support boxes (x0,x1,y0,y1 inclusive element
// ranges) + the boundary mask (em for curl, acoustic all rigid for div).
int ref_space(int kind, int degree, int elems, int levels, int64_t* n_full, int32_t* box,
              int64_t* mask, int64_t* nmask) {
  try {
    const rq::SpaceKind k = kind == 0 ? rq::SpaceKind::curl : rq::SpaceKind::divergence;
    const rq::VectorSpace vs = levels > 0
        ? rq::build_riga_space(k, degree, elems, levels, rq::BoxGeometry{})
        : rq::build_iga_space(k, degree, elems, rq::BoxGeometry{});
    *n_full = vs.N();
    if (box) {
      const rq::TensorSpace2D* comp[2] = {&vs.comp_x, &vs.comp_y};
      long g = 0;
      for (int c = 0; c < 2; ++c)
        for (int j = 0; j < comp[c]->ny(); ++j)
          for (int i = 0; i < comp[c]->nx(); ++i, ++g) {
            box[4 * g + 0] = comp[c]->sx.support_first_elem(i);
            box[4 * g + 1] = comp[c]->sx.support_last_elem(i);
            box[4 * g + 2] = comp[c]->sy.support_first_elem(j);
            box[4 * g + 3] = comp[c]->sy.support_last_elem(j);
          }
    }
    const auto m = rq::boundary_mask(vs, kind == 0 ? rq::ModelProblem::em : rq::ModelProblem::acoustic);
    *nmask = static_cast<int64_t>(m.size());
    if (mask)
      for (size_t i = 0; i < m.size(); ++i) mask[i] = m[i];
    return 0;
  } catch (const rq::Error& e) {
    return static_cast<int>(e.code());
  }
}

const char* ref_kern_backend() { return rq::kern::active().name; }

void ref_kern_spmv(int64_t n, const int64_t* rp, const int32_t* col, const double* val_c,
                   const double* x_c, double* y_c) {
  rq::kern::spmv_csr(n, rp, col, reinterpret_cast<const rq::cdouble*>(val_c),
                     reinterpret_cast<const rq::cdouble*>(x_c), reinterpret_cast<rq::cdouble*>(y_c));
}

void ref_kern_dotc(const double* x_c, const double* y_c, int64_t n, double* out_c) {
  const rq::cdouble r = rq::kern::dotc(reinterpret_cast<const rq::cdouble*>(x_c),
                                       reinterpret_cast<const rq::cdouble*>(y_c), n);
  out_c[0] = r.real();
  out_c[1] = r.imag();
}

uint64_t ref_kern_elim(double* tile_c, int64_t ld, const double* lcol_c, const double* urow_c,
                       int64_t rows, int64_t cols) {
  return rq::kern::active().elim_step(reinterpret_cast<rq::cdouble*>(tile_c), ld,
                                      reinterpret_cast<const rq::cdouble*>(lcol_c),
                                      reinterpret_cast<const rq::cdouble*>(urow_c), rows, cols);
}

int ref_select_backend(const char* name) {
  try {
    rq::kern::select_backend(name);
    return 0;
  } catch (const rq::Error& e) {
    return static_cast<int>(e.code());
  }
}

// Matrix Market through the reference's own sparse module (sparse.cpp:121-174).
int ref_mm_write(int64_t n, const int64_t* rowptr, const int32_t* col, const double* re, const double* im,
                 const char* path) {
  try {
    rq::SparseMatrix a;
    a.n = n;
    a.rowptr.assign(rowptr, rowptr + n + 1);
    a.col.assign(col, col + rowptr[n]);
    a.val.resize(rowptr[n]);
    for (int64_t k = 0; k < rowptr[n]; ++k) a.val[k] = rq::cdouble(re[k], im ? im[k] : 0.0);
    rq::write_matrix_market(a, path);
    return 0;
  } catch (const rq::Error& e) {
    return static_cast<int>(e.code());
  }
}

int ref_mm_write_vector(int64_t n, const double* re, const double* im, const char* path) {
  try {
    std::vector<rq::cdouble> x(n);
    for (int64_t i = 0; i < n; ++i) x[i] = rq::cdouble(re[i], im ? im[i] : 0.0);
    rq::write_matrix_market_vector(x, path);
    return 0;
  } catch (const rq::Error& e) {
    return static_cast<int>(e.code());
  }
}

// two calls: arrays NULL -> sizes; then the CSR (re / im split)
int ref_mm_read(const char* path, int64_t* n, int64_t* nnz, int64_t* rowptr, int32_t* col, double* re,
                double* im) {
  try {
    const rq::SparseMatrix a = rq::read_matrix_market(path);
    *n = a.n;
    *nnz = a.nnz();
    if (rowptr)
      for (size_t i = 0; i < a.rowptr.size(); ++i) rowptr[i] = a.rowptr[i];
    if (col)
      for (int64_t k = 0; k < a.nnz(); ++k) col[k] = a.col[k];
    if (re)
      for (int64_t k = 0; k < a.nnz(); ++k) re[k] = a.val[k].real(), im[k] = a.val[k].imag();
    return 0;
  } catch (const rq::Error& e) {
    return static_cast<int>(e.code());
  }
}

}  // extern "C"
