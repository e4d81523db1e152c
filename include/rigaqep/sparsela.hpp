// SPDX-License-Identifier: Apache-2.0
// sparsela drop-in for the reference tree: the SPEC
// signatures over the reference's own types (rq::SparseMatrix, rq::CostLedger,
// rq::VectorSpace, rq::Error — proj/include/rigaqep/{sparse,spaces,types}.hpp),
// implemented inline on top of the B200 C-ABI (include/rq_b200.h). A reference
// build adds this directory to its include path and links librq_b200.so
// (INTEGRATION.md). The GPU path is real FP64: complex matrices fail with
// errc::config (no CPU fallback); a complex right-hand side is solved as two
// real solves and charged as the one solve the reference performs.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "rigaqep/sparse.hpp"
#include "rigaqep/spaces.hpp"
#include "rigaqep/types.hpp"
#include "rq_b200.h"

namespace rq {

namespace b200 {
inline void check(int rc) {
  if (rc != 0) fail(static_cast<errc>(rc), std::string("rq_b200: ") + rq_last_error());
}
}  // namespace b200

/// Ordering: permutation + front structure handle.
struct Ordering {
  std::vector<std::int32_t> perm;  // perm[new] = old (free DOFs)
  std::string method = "geometric-nested-dissection";
  std::shared_ptr<rq_symbolic_t> sym;
  std::vector<std::int32_t> box;  // support boxes (n x 4) the ordering was built from
  int elems = 1, leaf = 64;
  long n() const { return static_cast<long>(perm.size()); }
};

namespace b200 {
inline Ordering ordering_from_boxes(std::int64_t n, const std::vector<std::int32_t>& box, int elems, int leaf,
                                    const char* method) {
  rq_symbolic_t* s = nullptr;
  check(rq_nd_order(n, box.data(), elems, leaf, &s));
  Ordering o;
  o.sym.reset(s, rq_symbolic_destroy);
  o.perm.resize(n);
  o.method = method;
  o.box = box;
  o.elems = elems;
  o.leaf = leaf;
  check(rq_symbolic_perm(s, o.perm.data()));
  return o;
}
/// sum over fronts and pivots of (nf - k - 1)^2: the factorization's
/// multiply-adds counted from the structure
inline double fa_macs(const Ordering& o) {
  rq_symbolic_stats st{};
  check(rq_symbolic_stats_get(o.sym.get(), &st));
  std::vector<std::int32_t> np(st.nfronts), nf(st.nfronts);
  check(rq_symbolic_fronts(o.sym.get(), nullptr, np.data(), nf.data(), nullptr, nullptr));
  double m = 0;
  for (std::size_t f = 0; f < np.size(); ++f)
    for (int k = 0; k < np[f]; ++k) m += static_cast<double>(nf[f] - k - 1) * (nf[f] - k - 1);
  return m;
}
/// per real solve: sum np^2 + 2 np (nf - np) (the stored L and U entries read)
inline double fb_macs(const Ordering& o) {
  rq_symbolic_stats st{};
  check(rq_symbolic_stats_get(o.sym.get(), &st));
  std::vector<std::int32_t> np(st.nfronts), nf(st.nfronts);
  check(rq_symbolic_fronts(o.sym.get(), nullptr, np.data(), nf.data(), nullptr, nullptr));
  double m = 0;
  for (std::size_t f = 0; f < np.size(); ++f) m += double(np[f]) * np[f] + 2.0 * np[f] * (nf[f] - np[f]);
  return m;
}
}  // namespace b200

/// nested_dissection_order(space): geometric ND over the
/// support boxes of the free DOFs (constrained = sorted eliminated DOF ids,
/// boundary_mask). Errors: none beyond the reference space's own.
inline Ordering nested_dissection_order(const VectorSpace& vs, const std::vector<long>& constrained,
                                        int leaf = 64) {
  std::vector<std::int32_t> box;
  const TensorSpace2D* comp[2] = {&vs.comp_x, &vs.comp_y};
  long g = 0;
  std::size_t ci = 0;
  for (int c = 0; c < 2; ++c)
    for (int j = 0; j < comp[c]->ny(); ++j)
      for (int i = 0; i < comp[c]->nx(); ++i, ++g) {
        if (ci < constrained.size() && constrained[ci] == g) {
          ++ci;
          continue;
        }
        box.push_back(comp[c]->sx.support_first_elem(i));
        box.push_back(comp[c]->sx.support_last_elem(i));
        box.push_back(comp[c]->sy.support_first_elem(j));
        box.push_back(comp[c]->sy.support_last_elem(j));
      }
  return b200::ordering_from_boxes(static_cast<std::int64_t>(box.size() / 4), box, vs.elems, leaf,
                                   "geometric-nested-dissection");
}

/// The "natural" Ordering of SPEC.md:110 (one dense front): for small
/// matrices without a space (SPEC's hand examples).
inline Ordering natural_order(long n) {
  return b200::ordering_from_boxes(n, std::vector<std::int32_t>(4 * static_cast<std::size_t>(n), 0), 1,
                                   static_cast<int>(n), "natural");
}

/// Factorization: immutable and device resident. Concurrent
/// solves on one factorization are safe: the library serialises
/// the calls that share its stream and solve buffers.
struct Factorization {
  std::shared_ptr<rq_factor_t> f;
  long n = 0;
  bool complex_values = false;  // factored as the real-equivalent 2n system
  std::int64_t nnz_l = 0, nnz_u = 0;
  double flops = 0;
  double fb_macs = 0;
};

inline std::vector<double> real_values(const SparseMatrix& a) {
  if (!a.is_real()) fail(errc::config, "the B200 path factors real matrices only");
  std::vector<double> v(a.val.size());
  for (std::size_t k = 0; k < v.size(); ++k) v[k] = a.val[k].real();
  return v;
}

/// lu_factorize: fa += the structural multiply-add count.
/// A complex A (a complex shift) is factored on the GPU as its
/// real-equivalent 2n system over the ordering's boxes repeated per (Re, Im)
/// pair (rq_factor_create_complex); the ledger charges the complex problem's
/// structural count of the given ordering, as the reference path would.
inline Factorization lu_factorize(const SparseMatrix& A, const Ordering& ord, CostLedger* ledger) {
  if (A.n != ord.n()) fail(errc::dimension, "lu_factorize: matrix and ordering sizes differ");
  rq_factor_t* f = nullptr;
  const bool cplx = !A.is_real();
  if (cplx) {
    if (ord.box.size() != 4 * static_cast<std::size_t>(A.n)) fail(errc::config, "ordering without support boxes");
    std::vector<std::int32_t> box2(8 * static_cast<std::size_t>(A.n));
    for (long k = 0; k < A.n; ++k)
      for (int t = 0; t < 4; ++t) box2[8 * k + t] = box2[8 * k + 4 + t] = ord.box[4 * k + t];
    const Ordering o2 = b200::ordering_from_boxes(2 * A.n, box2, ord.elems, ord.leaf, ord.method.c_str());
    std::vector<double> re(A.val.size()), im(A.val.size());
    for (std::size_t k = 0; k < re.size(); ++k) re[k] = A.val[k].real(), im[k] = A.val[k].imag();
    b200::check(rq_factor_create_complex(o2.sym.get(), A.n, A.rowptr.data(), A.col.data(), re.data(), im.data(), &f));
  } else {
    const std::vector<double> v = real_values(A);
    b200::check(rq_factor_create(ord.sym.get(), A.n, A.rowptr.data(), A.col.data(), v.data(), &f));
  }
  Factorization F;
  F.complex_values = cplx;
  F.f.reset(f, rq_factor_destroy);
  F.n = A.n;
  rq_symbolic_stats st{};
  b200::check(rq_symbolic_stats_get(ord.sym.get(), &st));
  F.nnz_l = st.nnz_l;
  F.nnz_u = st.nnz_u;
  F.flops = st.flops_lu;
  F.fb_macs = b200::fb_macs(ord);
  if (ledger) ledger->add_fa(static_cast<std::uint64_t>(b200::fa_macs(ord)));
  return F;
}

/// solve_factored: x = A^{-1} rhs; fb += one solve.
inline std::vector<cdouble> solve_factored(const Factorization& F, const std::vector<cdouble>& rhs,
                                           CostLedger* ledger) {
  if (static_cast<long>(rhs.size()) != F.n) fail(errc::dimension, "solve_factored dimension mismatch");
  if (F.complex_values) {  // cdouble[n] is the interleaved real-equivalent vector
    std::vector<cdouble> out(F.n);
    b200::check(rq_factor_solve_complex(F.f.get(), reinterpret_cast<const double*>(rhs.data()),
                                        reinterpret_cast<double*>(out.data()), 1));
    if (ledger) ledger->add_fb(static_cast<std::uint64_t>(F.fb_macs));
    return out;
  }
  bool cplx = false;
  for (const cdouble& z : rhs) cplx = cplx || z.imag() != 0.0;
  const int nr = cplx ? 2 : 1;
  std::vector<double> b(nr * F.n), x(nr * F.n);
  for (long i = 0; i < F.n; ++i) {
    b[i] = rhs[i].real();
    if (cplx) b[F.n + i] = rhs[i].imag();
  }
  b200::check(rq_factor_solve(F.f.get(), b.data(), x.data(), nr));
  std::vector<cdouble> out(F.n);
  for (long i = 0; i < F.n; ++i) out[i] = {x[i], cplx ? x[F.n + i] : 0.0};
  if (ledger) ledger->add_fb(static_cast<std::uint64_t>(F.fb_macs));
  return out;
}

}  // namespace rq
