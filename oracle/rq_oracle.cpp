// SPDX-License-Identifier: Apache-2.0
// ============================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY. CPU restatement of the reference path
// (arXiv 2112.14064 reference, /root/reference: proj/ sources + SPEC.md). Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load this library, and only as the checker or the timed
// CPU baseline. The product (paper_2112_14064_b200/) never calls it.
//
// Arithmetic is the reference's: complex double (types.hpp:11) through the
// six kern:: inner loops (kernels.hpp:17-39). Built two ways (oracle/Makefile):
//   liboracle.so                 kern:: restated here (kernels.cpp semantics)
//   _ref/liboracle_ref.so        -DORACLE_REF_KERN: kern:: calls go to the
//                                reference's own kernels.cpp/kernels_avx2.cpp
//                                compiled from /root/reference (patched
//                                elim_step declaration)
// The factor/solve/eigensolve layers do not exist in the reference; they are
// restated from SPEC.md (sparsela :279-378, eig :380-511) and PAPER.md
// (Alg. 2 :555-589). Parity pins: SPEC known answers, the paper's structural
// numbers, scipy dense eigensolves (tests/), and the reference kernels.
// ============================================================================
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include <omp.h>

#ifdef ORACLE_REF_KERN
#include "rigaqep/kernels.hpp"
#endif

using cd = std::complex<double>;

namespace oracle {

// ---------------------------------------------------------------------------
// kern:: (reference kernels.hpp:17-39)
#ifdef ORACLE_REF_KERN
inline void k_axpy(cd a, const cd* x, cd* y, size_t n) { rq::kern::axpy(a, x, y, n); }
inline cd k_dotc(const cd* x, const cd* y, size_t n) { return rq::kern::dotc(x, y, n); }
inline void k_scal(cd a, cd* x, size_t n) { rq::kern::scal(a, x, n); }
inline void k_spmv(size_t n, const int64_t* rp, const int32_t* col, const cd* val, const cd* x, cd* y) {
  rq::kern::spmv_csr(n, rp, col, val, x, y);
}
inline uint64_t k_elim(cd* tile, size_t ld, const cd* lcol, const cd* urow, size_t rows, size_t cols) {
  return rq::kern::active().elim_step(tile, ld, lcol, urow, rows, cols);
}
#else
// kernels.cpp:19-21
inline void k_axpy(cd a, const cd* x, cd* y, size_t n) {
  for (size_t i = 0; i < n; ++i) y[i] += a * x[i];
}
// kernels.cpp:23-32: conj(x) . y with split real accumulators
inline cd k_dotc(const cd* x, const cd* y, size_t n) {
  double rr = 0.0, ri = 0.0;
  for (size_t i = 0; i < n; ++i) {
    rr += x[i].real() * y[i].real() + x[i].imag() * y[i].imag();
    ri += x[i].real() * y[i].imag() - x[i].imag() * y[i].real();
  }
  return {rr, ri};
}
// kernels.cpp:34-36
inline void k_scal(cd a, cd* x, size_t n) {
  for (size_t i = 0; i < n; ++i) x[i] *= a;
}
// kernels.cpp:44-56: row loop, sequential accumulation
inline void k_spmv(size_t n, const int64_t* rp, const int32_t* col, const cd* val, const cd* x, cd* y) {
  for (size_t r = 0; r < n; ++r) {
    double ar = 0.0, ai = 0.0;
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
      const cd v = val[k], xc = x[col[k]];
      ar += v.real() * xc.real() - v.imag() * xc.imag();
      ai += v.real() * xc.imag() + v.imag() * xc.real();
    }
    y[r] = {ar, ai};
  }
}
// kernels.cpp:58-69 (rank1_update_scalar): rows with zero multiplier skipped
inline uint64_t k_elim(cd* tile, size_t ld, const cd* lcol, const cd* urow, size_t rows, size_t cols) {
  uint64_t macs = 0;
  for (size_t i = 0; i < rows; ++i) {
    const cd l = lcol[i];
    if (l == cd{}) continue;
    cd* row = tile + i * ld;
    for (size_t k = 0; k < cols; ++k) row[k] -= l * urow[k];
    macs += cols;
  }
  return macs;
}
#endif

// ---------------------------------------------------------------------------
// CostLedger (sparse.hpp:57-103), 8 flops per complex MAC
struct Ledger {
  uint64_t ops[6] = {0, 0, 0, 0, 0, 0};   // fa fb mv vv check restart
  double macs[6] = {0, 0, 0, 0, 0, 0};
  void add(int c, double m) { ops[c] += 1, macs[c] += m; }
};
enum { FA = 0, FB = 1, MV = 2, VV = 3, CHK = 4, RST = 5 };

struct Csr {
  int64_t n = 0;
  std::vector<int64_t> rp;
  std::vector<int32_t> col;
  std::vector<cd> val;
};

// rq::spmv / dot / axpy (sparse.cpp:59-72): ledger-charging wrappers
// Row chunks of kern::spmv_csr in parallel: each row's sum is the kernel's
// own sequential accumulation, so y is bit-identical for any thread count.
void spmv(const Csr& A, const cd* x, cd* y, Ledger* L) {
  const int64_t n = A.n, chunk = 4096;
  if (omp_get_max_threads() == 1 || n < 2 * chunk) {
    k_spmv(n, A.rp.data(), A.col.data(), A.val.data(), x, y);
  } else {
#pragma omp parallel for schedule(static)
    for (int64_t r0 = 0; r0 < n; r0 += chunk)
      k_spmv(std::min(chunk, n - r0), A.rp.data() + r0, A.col.data(), A.val.data(), x, y + r0);
  }
  if (L) L->add(MV, static_cast<double>(A.rp[A.n]));
}
cd dot(const cd* x, const cd* y, size_t n, Ledger* L) {
  if (L) L->add(VV, n);
  return k_dotc(x, y, n);
}
void axpy(cd a, const cd* x, cd* y, size_t n, Ledger* L) {
  if (L) L->add(VV, n);
  k_axpy(a, x, y, n);
}
// CGS projections over a basis: h_i = dot(V_i, w) for i < k (one kern::dotc
// per basis vector, vectors in parallel), then r -= sum_i h_i V_i as k
// kern::axpy calls in basis order over row chunks in parallel. Same
// arithmetic per entry as the sequential loops; charges k vv ops each.
void dots(const std::vector<std::vector<cd>>& V, int k, const cd* w, size_t n, cd* h, Ledger* L) {
#pragma omp parallel for schedule(dynamic, 1) if (k > 1)
  for (int i = 0; i < k; ++i) h[i] = k_dotc(V[i].data(), w, n);
  if (L)
    for (int i = 0; i < k; ++i) L->add(VV, n);
}
void axpys(const std::vector<std::vector<cd>>& V, int k, const cd* h, cd* r, size_t n, double sign, Ledger* L) {
  const size_t chunk = 8192;
#pragma omp parallel for schedule(static) if (n > 2 * chunk)
  for (size_t r0 = 0; r0 < n; r0 += chunk) {
    const size_t len = std::min(chunk, n - r0);
    for (int i = 0; i < k; ++i) k_axpy(sign * h[i], V[i].data() + r0, r + r0, len);
  }
  if (L)
    for (int i = 0; i < k; ++i) L->add(VV, n);
}

// ---------------------------------------------------------------------------
// nested_dissection_order
struct NDNode {
  int bx0, bx1, by0, by1;
  std::vector<int32_t> piv;
  std::vector<int> kids;
};

struct ND {
  const int32_t* box;
  int leaf;
  std::vector<NDNode> nodes;
  int rec(int x0, int x1, int y0, int y1, std::vector<int32_t> d) {
    const int w = x1 - x0, h = y1 - y0;
    if (static_cast<int>(d.size()) <= leaf || (w < 2 && h < 2)) {
      std::sort(d.begin(), d.end());
      nodes.push_back({x0, x1, y0, y1, d, {}});
      return static_cast<int>(nodes.size()) - 1;
    }
    const bool vx = w >= h;  // ties: vertical separator (cut x) first
    const int mid = vx ? x0 + w / 2 : y0 + h / 2;
    std::vector<int32_t> L, R, S;
    for (int32_t i : d) {
      const int a = box[4 * i + (vx ? 0 : 2)], b = box[4 * i + (vx ? 1 : 3)];
      (b < mid ? L : (a >= mid ? R : S)).push_back(i);
    }
    std::vector<int> kids;
    if (!L.empty()) kids.push_back(vx ? rec(x0, mid, y0, y1, L) : rec(x0, x1, y0, mid, L));
    if (!R.empty()) kids.push_back(vx ? rec(mid, x1, y0, y1, R) : rec(x0, x1, mid, y1, R));
    if (S.empty() && kids.size() == 1) return kids[0];
    std::sort(S.begin(), S.end());
    nodes.push_back({x0, x1, y0, y1, S, kids});
    return static_cast<int>(nodes.size()) - 1;
  }
};

// Front structure from the elimination tree (independent of the product's
// geometric rule): struct(j) = adj(j) ∩ {>j} ∪ struct(children) \ {j};
// one front per ND node with CB = ∪ struct(j) over its columns, minus pivots.
struct Symbolic {
  int64_t n = 0;
  std::vector<int32_t> perm, iperm;
  std::vector<int32_t> node_start, node_npiv, node_parent;
  std::vector<std::vector<int32_t>> node_rows;  // pivots then CB rows (new ids, ascending)
  std::vector<int32_t> etree;
  int64_t struct_nnz_l = 0;  // exact structural nnz(L) incl. diagonal
};

Symbolic symbolic(int64_t n, const int64_t* rp, const int32_t* col, const int32_t* box, int elems,
                  int leaf) {
  ND nd{box, leaf, {}};
  std::vector<int32_t> all(n);
  std::iota(all.begin(), all.end(), 0);
  nd.rec(0, elems, 0, elems, all);
  Symbolic S;
  S.n = n;
  const int nn = static_cast<int>(nd.nodes.size());
  S.node_parent.assign(nn, -1);
  for (int f = 0; f < nn; ++f) {
    S.node_start.push_back(static_cast<int32_t>(S.perm.size()));
    S.node_npiv.push_back(static_cast<int32_t>(nd.nodes[f].piv.size()));
    for (int32_t d : nd.nodes[f].piv) S.perm.push_back(d);
    for (int k : nd.nodes[f].kids) S.node_parent[k] = f;
  }
  S.iperm.assign(n, 0);
  for (int64_t i = 0; i < n; ++i) S.iperm[S.perm[i]] = static_cast<int32_t>(i);
  // column structures of L in the new order (symmetric pattern)
  std::vector<std::vector<int32_t>> st(n);
  S.etree.assign(n, -1);
  std::vector<std::vector<int32_t>> kids(n);
  for (int64_t j = 0; j < n; ++j) {
    std::vector<int32_t> s;
    const int32_t old = S.perm[j];
    for (int64_t k = rp[old]; k < rp[old + 1]; ++k) {
      const int32_t i = S.iperm[col[k]];
      if (i > j) s.push_back(i);
    }
    for (int32_t c : kids[j])
      for (int32_t i : st[c])
        if (i > j) s.push_back(i);
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
    if (!s.empty()) {
      S.etree[j] = s[0];
      kids[s[0]].push_back(static_cast<int32_t>(j));
    }
    S.struct_nnz_l += 1 + static_cast<int64_t>(s.size());
    st[j] = std::move(s);
  }
  S.node_rows.resize(nn);
  for (int f = 0; f < nn; ++f) {
    const int32_t s0 = S.node_start[f], e0 = s0 + S.node_npiv[f];
    std::vector<int32_t> rows;
    for (int32_t j = s0; j < e0; ++j)
      for (int32_t i : st[j])
        if (i >= e0) rows.push_back(i);
    std::sort(rows.begin(), rows.end());
    rows.erase(std::unique(rows.begin(), rows.end()), rows.end());
    std::vector<int32_t> all_rows;
    for (int32_t j = s0; j < e0; ++j) all_rows.push_back(j);
    all_rows.insert(all_rows.end(), rows.begin(), rows.end());
    S.node_rows[f] = std::move(all_rows);
  }
  // Rows of an empty-separator node are its children's CB rows (pass-through).
  for (int f = 0; f < nn; ++f) {
    if (S.node_npiv[f] != 0) continue;
    std::vector<int32_t> rows;
    for (int k : nd.nodes[f].kids) {
      const auto& kr = S.node_rows[k];
      rows.insert(rows.end(), kr.begin() + S.node_npiv[k], kr.end());
    }
    std::sort(rows.begin(), rows.end());
    rows.erase(std::unique(rows.begin(), rows.end()), rows.end());
    S.node_rows[f] = rows;
  }
  return S;
}

// ---------------------------------------------------------------------------
// lu_factorize: multifrontal, row-major dense
// fronts, threshold u = 0.1 partial pivoting among fully-summed rows, prefer
// the diagonal, ties -> lowest index, singular if max candidate < 1e-300.
struct FrontF {
  int32_t npiv = 0, nf = 0;
  std::vector<int32_t> rows;
  std::vector<cd> F;        // nf x nf row-major while the front is live: L\U and its CB
  std::vector<cd> U, Lc;    // after the parent consumed the CB: rows 0..npiv-1 (npiv x nf)
                            // and rows npiv..nf-1 of columns 0..npiv-1 ((nf-npiv) x npiv)
  std::vector<int32_t> ipiv;
  int64_t swaps = 0;
  uint64_t macs = 0;
  bool compacted = false;
  // L\U entry (i, c) with i < npiv or c < npiv
  cd lu(int i, int c) const {
    if (!compacted) return F[static_cast<size_t>(i) * nf + c];
    return i < npiv ? U[static_cast<size_t>(i) * nf + c] : Lc[static_cast<size_t>(i - npiv) * npiv + c];
  }
  void compact() {
    if (compacted) return;
    U.assign(F.begin(), F.begin() + static_cast<size_t>(npiv) * nf);
    Lc.resize(static_cast<size_t>(nf - npiv) * npiv);
    for (int i = npiv; i < nf; ++i)
      std::copy(F.begin() + static_cast<size_t>(i) * nf, F.begin() + static_cast<size_t>(i) * nf + npiv,
                Lc.begin() + static_cast<size_t>(i - npiv) * npiv);
    std::vector<cd>().swap(F);
    compacted = true;
  }
};

struct Factor {
  const Symbolic* S = nullptr;
  std::vector<FrontF> fr;
  int64_t swaps = 0;
  double fa_macs = 0;
  double fb_macs = 0;  // per solve
};

struct OracleError {
  int code;
  std::string msg;
};

// Factor one front: assemble the original entries and the children's
// contribution blocks (extend-add, children in ascending order), then
// right-looking threshold-pivoted elimination with kern::elim_step. Rows of a
// rank-1 step are independent (each row scales its multiplier, then
// row -= l * urow), so large trailing blocks split into row chunks executed as
// OpenMP tasks: every entry sees the same operations in the same order, the
// factors are bit-identical for any thread count (SPEC.md:366 allows concurrent
// subtree factorization).
void factor_front(Factor& R, int f, const std::vector<std::vector<std::pair<int64_t, cd>>>& orig,
                  const std::vector<std::vector<int>>& kids) {
  const Symbolic& S = *R.S;
  FrontF& Fr = R.fr[f];
  Fr.rows = S.node_rows[f];
  Fr.nf = static_cast<int32_t>(Fr.rows.size());
  Fr.npiv = S.node_npiv[f];
  const int nf = Fr.nf, np = Fr.npiv;
  Fr.F.assign(static_cast<size_t>(nf) * nf, cd{});
  auto loc = [&](int32_t g) {
    const auto it = std::lower_bound(Fr.rows.begin(), Fr.rows.end(), g);
    if (it == Fr.rows.end() || *it != g) throw OracleError{7, "entry outside front"};
    return static_cast<int>(it - Fr.rows.begin());
  };
  for (auto& e : orig[f]) {
    const int r = loc(static_cast<int32_t>(e.first / S.n)), c = loc(static_cast<int32_t>(e.first % S.n));
    Fr.F[static_cast<size_t>(r) * nf + c] += e.second;
  }
  for (int c : kids[f]) {  // extend-add
    FrontF& K = R.fr[c];
    const int knp = K.npiv, knf = K.nf;
    std::vector<int> map(knf - knp);
    for (int t = knp; t < knf; ++t) map[t - knp] = loc(K.rows[t]);
    for (int a = knp; a < knf; ++a)
      for (int b = knp; b < knf; ++b)
        Fr.F[static_cast<size_t>(map[a - knp]) * nf + map[b - knp]] += K.F[static_cast<size_t>(a) * knf + b];
    K.compact();  // the child's CB is consumed
  }
  Fr.ipiv.assign(np, 0);
  std::vector<cd> lcol(nf);
  for (int k = 0; k < np; ++k) {
    double best = -1.0;
    int bi = k;
    for (int i = k; i < np; ++i) {
      const double v = std::abs(Fr.F[static_cast<size_t>(i) * nf + k]);
      if (v > best) best = v, bi = i;
    }
    if (!(best >= 1e-300)) throw OracleError{8, "singular pivot block"};
    const double diag = std::abs(Fr.F[static_cast<size_t>(k) * nf + k]);
    const int p = diag >= 0.1 * best ? k : bi;
    Fr.ipiv[k] = p;
    if (p != k) {
      ++Fr.swaps;
      for (int c = 0; c < nf; ++c)
        std::swap(Fr.F[static_cast<size_t>(k) * nf + c], Fr.F[static_cast<size_t>(p) * nf + c]);
    }
    const cd piv = Fr.F[static_cast<size_t>(k) * nf + k];
    const int rows = nf - k - 1, cols = nf - k - 1;
    cd* F = Fr.F.data();
    cd* lc = lcol.data();
    auto chunk = [F, lc, piv, k, nf, cols](int r0, int r1) -> uint64_t {
      for (int i = k + 1 + r0; i < k + 1 + r1; ++i) {
        cd& a = F[static_cast<size_t>(i) * nf + k];
        a /= piv;
        lc[i - k - 1] = a;
      }
      return k_elim(&F[static_cast<size_t>(k + 1 + r0) * nf + k + 1], nf, lc + r0,
                    &F[static_cast<size_t>(k) * nf + k + 1], r1 - r0, cols);
    };
    const int64_t work = static_cast<int64_t>(rows) * cols;
    if (work < (int64_t{1} << 17) || omp_get_num_threads() == 1) {
      Fr.macs += chunk(0, rows);
    } else {
      const int g = 32;
      uint64_t m = 0;
#pragma omp taskloop grainsize(1) reduction(+ : m)
      for (int b = 0; b < (rows + g - 1) / g; ++b) m += chunk(b * g, std::min(rows, (b + 1) * g));
      Fr.macs += m;
    }
  }
}

void factor_subtree(Factor& R, int f, const std::vector<std::vector<std::pair<int64_t, cd>>>& orig,
                    const std::vector<std::vector<int>>& kids) {
  for (int c : kids[f]) {
#pragma omp task default(shared) firstprivate(c)
    factor_subtree(R, c, orig, kids);
  }
#pragma omp taskwait
  factor_front(R, f, orig, kids);
}

Factor lu_factorize(const Symbolic& S, const Csr& A, Ledger* L) {
  Factor R;
  R.S = &S;
  const int nn = static_cast<int>(S.node_rows.size());
  R.fr.resize(nn);
  std::vector<std::vector<int>> kids(nn);
  std::vector<int> roots;
  for (int f = 0; f < nn; ++f)
    if (S.node_parent[f] >= 0)
      kids[S.node_parent[f]].push_back(f);
    else
      roots.push_back(f);
  std::vector<int32_t> owner(S.n);
  for (int f = 0; f < nn; ++f)
    for (int k = 0; k < S.node_npiv[f]; ++k) owner[S.node_start[f] + k] = f;
  // original entries per owning front
  std::vector<std::vector<std::pair<int64_t, cd>>> orig(nn);  // (packed r*n+c new ids, value)
  for (int64_t i = 0; i < A.n; ++i)
    for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) {
      const int64_t r = S.iperm[i], c = S.iperm[A.col[k]];
      orig[owner[std::min(r, c)]].push_back({r * S.n + c, A.val[k]});
    }
  std::string err;
  int err_code = 0;
#pragma omp parallel
#pragma omp single
  {
    for (int r : roots) {
#pragma omp task default(shared) firstprivate(r)
      {
        try {
          factor_subtree(R, r, orig, kids);
        } catch (const OracleError& e) {
#pragma omp critical
          if (!err_code) err_code = e.code, err = e.msg;
        }
      }
    }
  }
  if (err_code) throw OracleError{err_code, err};
  uint64_t macs = 0;
  for (int f = 0; f < nn; ++f) {
    R.fr[f].compact();
    macs += R.fr[f].macs;
    R.swaps += R.fr[f].swaps;
    const double np = R.fr[f].npiv, nf = R.fr[f].nf;
    R.fb_macs += np * np + 2.0 * np * (nf - np);
  }
  R.fa_macs = static_cast<double>(macs);
  // the ledger counts multiply-adds analytically from the front structure
  // (SPEC.md:376): sum over pivots of (nf-k-1)^2, the dense rank-1 updates
  // (R.fa_macs is the kernel-returned count, which skips zero multipliers)
  double fa = 0;
  for (int f = 0; f < nn; ++f)
    for (int k = 0; k < R.fr[f].npiv; ++k) {
      const double r = R.fr[f].nf - k - 1.0;
      fa += r * r;
    }
  if (L) L->add(FA, fa);
  return R;
}

// solve_factored: permute, L solve, U solve (original order).
// Row-oriented traversal of the stored L\U (contiguous rows): each y entry
// receives its updates in the same (ascending pivot) order as the
// column-oriented substitution, so the result is the same bit for bit; the
// contribution rows of a front are independent and run in parallel.
// a * b for finite operands: the value std::complex's operator* returns
// (re = ac - bd, im = ad + bc, no contraction) without the __muldc3
// inf/nan-recovery call
inline cd cmul(cd a, cd b) {
  return {a.real() * b.real() - a.imag() * b.imag(), a.real() * b.imag() + a.imag() * b.real()};
}

void solve_factored(const Factor& R, const cd* b, cd* x, Ledger* L) {
  const Symbolic& S = *R.S;
  const int nn = static_cast<int>(R.fr.size());
  std::vector<cd> y(S.n);
  for (int64_t i = 0; i < S.n; ++i) y[i] = b[S.perm[i]];
  // forward: y[rows] of each front updated in postorder
  for (int f = 0; f < nn; ++f) {
    const FrontF& Fr = R.fr[f];
    const int nf = Fr.nf, np = Fr.npiv;
    for (int k = 0; k < np; ++k) {
      const int p = Fr.ipiv[k];
      if (p != k) std::swap(y[Fr.rows[k]], y[Fr.rows[p]]);
    }
    for (int i = 1; i < np; ++i) {
      cd s = y[Fr.rows[i]];
      for (int k = 0; k < i; ++k) s -= cmul(Fr.lu(i, k), y[Fr.rows[k]]);
      y[Fr.rows[i]] = s;
    }
    auto cb_row = [&](int i) {
      cd s = y[Fr.rows[i]];
      for (int k = 0; k < np; ++k) s -= cmul(Fr.lu(i, k), y[Fr.rows[k]]);
      y[Fr.rows[i]] = s;
    };
    if (static_cast<int64_t>(nf - np) * np > (1 << 16) && omp_get_max_threads() > 1) {
#pragma omp parallel for schedule(static)
      for (int i = np; i < nf; ++i) cb_row(i);
    } else {
      for (int i = np; i < nf; ++i) cb_row(i);
    }
  }
  // backward, reverse postorder
  for (int f = nn - 1; f >= 0; --f) {
    const FrontF& Fr = R.fr[f];
    const int nf = Fr.nf, np = Fr.npiv;
    for (int k = np - 1; k >= 0; --k) {
      cd s = y[Fr.rows[k]];
      for (int c = k + 1; c < nf; ++c) s -= cmul(Fr.lu(k, c), y[Fr.rows[c]]);
      y[Fr.rows[k]] = s / Fr.lu(k, k);
    }
  }
  for (int64_t i = 0; i < S.n; ++i) x[S.perm[i]] = y[i];
  if (L) L->add(FB, R.fb_macs);
}

// ---------------------------------------------------------------------------
// Dense complex Schur (m x m, column-major) for ritz_extract/restart
// (SPEC.md:444-461): Hessenberg by Givens, shifted QR, Givens reordering.
struct DM {
  int n;
  std::vector<cd> a;
  explicit DM(int n_ = 0) : n(n_), a(static_cast<size_t>(n_) * n_) {}
  cd& operator()(int i, int j) { return a[i + static_cast<size_t>(j) * n]; }
};

void rot(cd f, cd g, double& c, cd& s) {
  const double af = std::abs(f), ag = std::abs(g);
  if (ag == 0) { c = 1; s = 0; return; }
  if (af == 0) { c = 0; s = std::conj(g) / ag; return; }
  const double r = std::sqrt(af * af + ag * ag);
  c = af / r;
  s = f / af * std::conj(g) / r;
}
// left: rows (i, i+1) <- G rows; right: cols (j, j+1) <- cols G^H
void lrot(DM& A, int i, int c0, double c, cd s) {
  for (int j = c0; j < A.n; ++j) {
    const cd x = A(i, j), y = A(i + 1, j);
    A(i, j) = c * x + s * y;
    A(i + 1, j) = c * y - std::conj(s) * x;
  }
}
void rrot(DM& A, int j, int r1, double c, cd s) {
  for (int i = 0; i < r1; ++i) {
    const cd x = A(i, j), y = A(i, j + 1);
    A(i, j) = c * x + std::conj(s) * y;
    A(i, j + 1) = c * y - s * x;
  }
}

bool schur(DM& T, DM& Z) {
  const int n = T.n;
  Z = DM(n);
  for (int i = 0; i < n; ++i) Z(i, i) = 1;
  for (int k = 0; k + 2 < n; ++k)  // Hessenberg via Givens from the bottom
    for (int i = n - 1; i > k + 1; --i) {
      double c;
      cd s;
      rot(T(i - 1, k), T(i, k), c, s);
      lrot(T, i - 1, 0, c, s);
      rrot(T, i - 1, n, c, s);
      rrot(Z, i - 1, n, c, s);
      T(i, k) = 0;
    }
  const double eps = std::numeric_limits<double>::epsilon();
  int hi = n - 1, it = 0, tot = 0;
  while (hi > 0) {
    int l = hi;
    while (l > 0 && std::abs(T(l, l - 1)) > eps * (std::abs(T(l - 1, l - 1)) + std::abs(T(l, l)))) --l;
    if (l > 0) T(l, l - 1) = 0;
    if (l == hi) { --hi; it = 0; continue; }
    if (++tot > 30 * n) return false;
    ++it;
    cd mu;
    const cd a = T(hi - 1, hi - 1), b = T(hi - 1, hi), c2 = T(hi, hi - 1), d = T(hi, hi);
    if (it % 10 == 0) {
      mu = d + std::abs(c2);
    } else {
      const cd tr2 = (a + d) / 2.0, dsc = std::sqrt((a - d) * (a - d) / 4.0 + b * c2);
      mu = std::abs(tr2 + dsc - d) < std::abs(tr2 - dsc - d) ? tr2 + dsc : tr2 - dsc;
    }
    for (int k = l; k < hi; ++k) {
      double c;
      cd s;
      if (k == l) rot(T(l, l) - mu, T(l + 1, l), c, s);
      else rot(T(k, k - 1), T(k + 1, k - 1), c, s);
      lrot(T, k, std::max(l, k - 1), c, s);
      if (k > l) T(k + 1, k - 1) = 0;
      rrot(T, k, std::min(k + 3, hi + 1), c, s);
      rrot(Z, k, n, c, s);
    }
  }
  return true;
}

void schur_move_front(DM& T, DM& Z, std::vector<int>& sel) {
  int ks = 0;
  for (int k = 0; k < T.n; ++k) {
    if (!sel[k]) continue;
    for (int j = k - 1; j >= ks; --j) {
      const cd a = T(j, j), b = T(j + 1, j + 1);
      double c;
      cd s;
      rot(T(j, j + 1), b - a, c, s);
      lrot(T, j, j + 2, c, s);
      rrot(T, j, j, c, s);
      T(j, j) = b;
      T(j + 1, j + 1) = a;
      rrot(Z, j, Z.n, c, s);
      std::swap(sel[j], sel[j + 1]);
    }
    ++ks;
  }
}

// ---------------------------------------------------------------------------
// Quadratic eigensolver: operator, B-inner, CGS2 Arnoldi,
// complex Krylov-Schur with the completeness guard of SURVEY.md §7 H1.
struct Pencil {
  Csr K, C, M;
  double nK = 0, nC = 0, nM = 0;  // 1-norms (sparse.cpp:38-45)
};

double norm1(const Csr& A) {
  std::vector<double> cs(A.n, 0.0);
  for (int64_t r = 0; r < A.n; ++r)
    for (int64_t k = A.rp[r]; k < A.rp[r + 1]; ++k) cs[A.col[k]] += std::abs(A.val[k]);
  return cs.empty() ? 0.0 : *std::max_element(cs.begin(), cs.end());
}

struct Operator {
  const Pencil* P;
  const Factor* F;
  cd s;
  int64_t n;
  std::vector<cd> t1, t2;
  // apply_operator: r_u = -Q(s)^{-1}(s M v_u + C v_u + M v_l); r_l = s r_u + v_u
  void apply(const cd* v, cd* r, Ledger* L) {
    t1.resize(n);
    t2.resize(n);
    spmv(P->C, v, t1.data(), L);              // C v_u
    spmv(P->M, v, t2.data(), L);              // M v_u
    axpy(s, t2.data(), t1.data(), n, L);      // + s M v_u
    spmv(P->M, v + n, t2.data(), L);          // M v_l
    axpy(1.0, t2.data(), t1.data(), n, L);    // + M v_l
    solve_factored(*F, t1.data(), r, L);
    k_scal(-1.0, r, n);
    for (int64_t i = 0; i < n; ++i) r[n + i] = v[i];
    axpy(s, r, r + n, n, L);
  }
  // b_inner: x_u^H y_u + x_l^H M y_l
  void bvec(const cd* y, cd* w, Ledger* L) {
    std::copy(y, y + n, w);
    spmv(P->M, y + n, w + n, L);
  }
};

uint64_t splitmix(uint64_t& x) {
  uint64_t z = (x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
double uni(uint64_t& s) { return (static_cast<double>(splitmix(s) >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0; }

struct EigOut {
  std::vector<cd> lam;
  std::vector<double> res;
  std::vector<std::vector<cd>> vec;
  int cycles = 0, guard = 0, nconv = 0;
  bool ok = false;
};

// Arnoldi steps j = k .. m-1 (Alg. 2 lines 7-13)
// with CGS2: r = S v_j; twice {w = B r; h = V_j^H w; r -= V_j h};
// h_{j+1,j} = ||r||_B, v_{j+1} = r / h_{j+1,j}. H accumulates both passes.
void arnoldi_steps(Operator& op, std::vector<std::vector<cd>>& V, DM& H, int k, int m, std::vector<cd>& r,
                   std::vector<cd>& w, Ledger* L) {
  const int64_t n2 = 2 * op.n;
  for (int j = k; j < m; ++j) {
    op.apply(V[j].data(), r.data(), L);
    for (int pass = 0; pass < 2; ++pass) {  // CGS2
      op.bvec(r.data(), w.data(), L);
      std::vector<cd> h(j + 1);
      dots(V, j + 1, w.data(), n2, h.data(), L);
      axpys(V, j + 1, h.data(), r.data(), n2, -1.0, L);
      for (int i = 0; i <= j; ++i) H(i, j) += h[i];
    }
    op.bvec(r.data(), w.data(), L);
    const double b = std::sqrt(std::max(0.0, dot(r.data(), w.data(), n2, L).real()));
    H(j + 1, j) = b;
    for (int64_t i = 0; i < n2; ++i) V[j + 1][i] = r[i] / b;
  }
}

// Block Arnoldi steps (block Krylov-Schur; the B200
// build's block mode, operation for operation): for kc = k, k+bs, ... while
// kc + bs <= m: R_b = S v_{kc+b} (b < bs); CGS2 of the block against V[0, kt),
// kt = kc + bs (per pass: w_b = B R_b for every member, then h_b = V^H w_b and
// R_b -= V h_b); then the block's own CGS2 (member b against V[kt, kt+b)) and
// B-normalisation into V[kt+b]. H(i, kc+b) accumulates the projections,
// H(kt+b, kc+b) = ||R_b||_B.
// Step plan (the B200 build's, eigs.cpp plan_steps): width bs while the cycle
// has room for at least min_steps such steps, else width 1 (banded block
// Arnoldi: S applied to the oldest frontier vector); a step of width wd
// applies S to V[kc, kc+wd), projects against V[0, kc+bs) and appends
// V[kc+bs, kc+bs+wd); the cycle ends at m accounted vectors.
void arnoldi_block_steps(Operator& op, std::vector<std::vector<cd>>& V, DM& H, int k, int m, int bs,
                         std::vector<std::vector<cd>>& R, std::vector<cd>& w, Ledger* L, int min_steps) {
  const int64_t n2 = 2 * op.n;
  const int wd0 = (m - k) >= bs * min_steps ? bs : 1;
  for (int kc = k; kc < m; kc += wd0) {
    const int wd = std::min(wd0, m - kc);
    const int kt = kc + bs;
    for (int b = 0; b < wd; ++b) op.apply(V[kc + b].data(), R[b].data(), L);
    if (wd == 1) {  // a width-1 step: the single-vector CGS2 step
      for (int pass = 0; pass < 2; ++pass) {
        op.bvec(R[0].data(), w.data(), L);
        std::vector<cd> h(kt);
        dots(V, kt, w.data(), n2, h.data(), L);
        axpys(V, kt, h.data(), R[0].data(), n2, -1.0, L);
        for (int i = 0; i < kt; ++i) H(i, kc) += h[i];
      }
      op.bvec(R[0].data(), w.data(), L);
      const double beta = std::sqrt(std::max(0.0, dot(R[0].data(), w.data(), n2, L).real()));
      H(kt, kc) = beta;
      for (int64_t i = 0; i < n2; ++i) V[kt][i] = R[0][i] / beta;
      continue;
    }
    // BCGS2: two passes of {project the block against V[0, kt), B-orthonormalise
    // it member by member (CGS2 against the earlier members)}; pass 2 works on
    // the normalised pass-1 block Q1: S V_blk = V (H1 + H2 R1) + Q2 R2 R1
    std::vector<std::vector<cd>> Hp(2, std::vector<cd>(static_cast<size_t>(kt) * wd, 0.0));
    std::vector<std::vector<cd>> Rq(2, std::vector<cd>(static_cast<size_t>(wd) * wd, 0.0));
    for (int pass = 0; pass < 2; ++pass) {
      std::vector<std::vector<cd>>& X = R;  // pass 0: R; pass 1: Q1 (copied back into R)
      std::vector<std::vector<cd>> h(wd, std::vector<cd>(kt));
      for (int b = 0; b < wd; ++b) {
        op.bvec(X[b].data(), w.data(), L);
        dots(V, kt, w.data(), n2, h[b].data(), L);
      }
      for (int b = 0; b < wd; ++b) {
        axpys(V, kt, h[b].data(), X[b].data(), n2, -1.0, L);
        for (int i = 0; i < kt; ++i) Hp[pass][i + static_cast<size_t>(b) * kt] = h[b][i];
      }
      for (int b = 0; b < wd; ++b) {
        for (int sub = 0; sub < 2 && b > 0; ++sub) {
          op.bvec(X[b].data(), w.data(), L);
          std::vector<cd> g(b);
          for (int i = 0; i < b; ++i) g[i] = dot(V[kt + i].data(), w.data(), n2, L);
          for (int i = 0; i < b; ++i) {
            axpy(-g[i], V[kt + i].data(), X[b].data(), n2, L);
            Rq[pass][i + static_cast<size_t>(b) * wd] += g[i];
          }
        }
        op.bvec(X[b].data(), w.data(), L);
        const double beta = std::sqrt(std::max(0.0, dot(X[b].data(), w.data(), n2, L).real()));
        Rq[pass][b + static_cast<size_t>(b) * wd] = beta;
        for (int64_t i = 0; i < n2; ++i) V[kt + b][i] = X[b][i] / beta;
      }
      if (pass == 0)
        for (int b = 0; b < wd; ++b) R[b] = V[kt + b];
    }
    for (int b = 0; b < wd; ++b) {
      for (int i = 0; i < kt; ++i) {
        cd v = Hp[0][i + static_cast<size_t>(b) * kt];
        for (int t = 0; t <= b; ++t) v += Hp[1][i + static_cast<size_t>(t) * kt] * Rq[0][t + static_cast<size_t>(b) * wd];
        H(i, kc + b) += v;
      }
      for (int i = 0; i <= b; ++i) {
        cd v = 0.0;
        for (int t = i; t <= b; ++t) v += Rq[1][i + static_cast<size_t>(t) * wd] * Rq[0][t + static_cast<size_t>(b) * wd];
        H(kt + i, kc + b) = v;
      }
    }
  }
}

// arnoldi_run: v1 B-normalised (one B-product, one dot),
// then m steps. V: m+1 vectors of 2n; H: (m+1) x m.
void arnoldi_run(Operator& op, const cd* v1, int m, std::vector<std::vector<cd>>& V, DM& H, Ledger* L) {
  const int64_t n2 = 2 * op.n;
  V.assign(m + 1, std::vector<cd>(n2));
  H = DM(m + 1);
  std::vector<cd> r(v1, v1 + n2), w(n2);
  op.bvec(r.data(), w.data(), L);
  const double b = std::sqrt(std::max(0.0, dot(r.data(), w.data(), n2, L).real()));
  for (int64_t i = 0; i < n2; ++i) V[0][i] = r[i] / b;
  arnoldi_steps(op, V, H, 0, m, r, w, L);
}

// bs > 1: block Krylov-Schur: a basis of m accounted
// vectors plus a frontier block of bs, steps of arnoldi_block_steps, the
// residual of a Ritz vector y is ||E y|| with E the bs rows of H below the
// accounted block, and a restart keeps the frontier block. Start / deflation
// blocks: member b from splitmix64(seed + b * golden) (b = 0: the
// single-vector start), CGS2 against everything before it.
EigOut solve_quadratic(Operator& op, int nev, int m, double tol, uint64_t seed, int max_restarts,
                       int guard_on, Ledger* L, int bs, int min_steps = 1) {
  const int64_t n = op.n, n2 = 2 * n;
  const double sig = op.s.real();
  const int keep_t = nev + std::min(20, m - nev - 1);
  std::vector<std::vector<cd>> V(m + bs, std::vector<cd>(n2)), V2 = V;
  std::vector<std::vector<cd>> R(bs, std::vector<cd>(n2));
  std::vector<cd> r(n2), w(n2);
  DM H(m + bs);  // (m+bs) x (m+bs), columns 0..m-1 used
  auto fresh_one = [&](uint64_t sd, int nlock, std::vector<cd>& dst) {
    uint64_t st = sd;
    for (int64_t i = 0; i < n2; ++i) r[i] = uni(st);
    for (int pass = 0; pass < 2 && nlock > 0; ++pass) {
      op.bvec(r.data(), w.data(), L);
      std::vector<cd> h(nlock);
      dots(V, nlock, w.data(), n2, h.data(), L);
      axpys(V, nlock, h.data(), r.data(), n2, -1.0, L);
    }
    op.bvec(r.data(), w.data(), L);
    const double b = std::sqrt(std::max(0.0, dot(r.data(), w.data(), n2, L).real()));
    for (int64_t i = 0; i < n2; ++i) dst[i] = r[i] / b;
  };
  auto fresh = [&](uint64_t sd, int nlock) {
    for (int b = 0; b < bs; ++b) fresh_one(sd + 0x9E3779B97F4A7C15ull * static_cast<uint64_t>(b), nlock + b, V[nlock + b]);
  };
  fresh(seed, 0);
  int k = 0, cycles = 0, gp = 0;
  EigOut out;
  std::vector<double> prev;
  int pass_cycles = 0;  // max_restarts bounds each pass (main + every guard pass)
  while (pass_cycles < max_restarts) {
    ++cycles;
    ++pass_cycles;
    const int mm = m, m0 = mm - bs;
    if (bs == 1)
      arnoldi_steps(op, V, H, k, m, r, w, L);
    else
      arnoldi_block_steps(op, V, H, k, m, bs, R, w, L, min_steps);
    DM T(mm), Z;
    for (int j = 0; j < mm; ++j)
      for (int i = 0; i < mm; ++i) T(i, j) = H(i, j);
    if (!schur(T, Z)) throw OracleError{4, "QR did not converge"};
    // eigenvectors of T, Ritz data
    std::vector<cd> th(mm), lam(mm);
    std::vector<double> est(mm);
    DM Y(mm);
    for (int j = 0; j < mm; ++j) {
      th[j] = T(j, j);
      lam[j] = op.s + 1.0 / th[j];
      Y(j, j) = 1;
      for (int i = j - 1; i >= 0; --i) {
        cd s = 0;
        for (int t = i + 1; t <= j; ++t) s += T(i, t) * Y(t, j);
        cd den = T(i, i) - th[j];
        if (std::abs(den) < 1e-300) den = 1e-300;
        Y(i, j) = -s / den;
      }
      double nr = 0;
      for (int i = 0; i <= j; ++i) nr += std::norm(Y(i, j));
      nr = std::sqrt(nr);
      for (int i = 0; i <= j; ++i) Y(i, j) /= nr;
      if (bs == 1) {
        cd yl = 0;
        for (int i = 0; i <= j; ++i) yl += Z(m - 1, i) * Y(i, j);
        est[j] = std::abs(H(m, m - 1) * yl) / std::abs(th[j]);
      } else {  // ||E y|| / |theta|, E = H(mm.., m0..mm)
        std::vector<cd> yl(bs, 0.0);
        for (int q = 0; q < bs; ++q)
          for (int i = 0; i <= j; ++i) yl[q] += Z(m0 + q, i) * Y(i, j);
        double e2 = 0;
        for (int a = 0; a < bs; ++a) {
          cd t = 0;
          for (int q = 0; q < bs; ++q) t += H(mm + a, m0 + q) * yl[q];
          e2 += std::norm(t);
        }
        est[j] = std::sqrt(e2) / std::abs(th[j]);
      }
    }
    std::vector<int> ord(mm);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) {
      const double da = std::abs(lam[a] - sig), db = std::abs(lam[b] - sig);
      if (da != db) return da < db;
      return lam[a].imag() > lam[b].imag();
    });
    std::vector<double> cres(nev, 1.0);
    std::vector<std::vector<cd>> cvec(nev);
    bool all = true;
    for (int c = 0; c < nev; ++c)
      if (!(est[ord[c]] <= 1e3 * tol)) all = false;
    if (all) {
      for (int c = 0; c < nev; ++c) {
        const int i = ord[c];
        std::vector<cd> y(mm, 0.0), x(n2, 0.0);
        for (int row = 0; row < mm; ++row)
          for (int t = 0; t <= i; ++t) y[row] += Z(row, t) * Y(t, i);
        axpys(V, mm, y.data(), x.data(), n2, 1.0, nullptr);
        const bool low = std::abs(lam[i]) > 1.0;  // larger-norm block
        std::vector<cd> u(x.begin() + (low ? n : 0), x.begin() + (low ? n2 : n));
        // explicit pencil residual
        std::vector<cd> a(n), q(n, 0.0);
        spmv(op.P->K, u.data(), a.data(), nullptr);
        for (int64_t e = 0; e < n; ++e) q[e] += a[e];
        spmv(op.P->C, u.data(), a.data(), nullptr);
        for (int64_t e = 0; e < n; ++e) q[e] += lam[i] * a[e];
        spmv(op.P->M, u.data(), a.data(), nullptr);
        for (int64_t e = 0; e < n; ++e) q[e] += lam[i] * lam[i] * a[e];
        if (L) L->add(CHK, 3.0 * op.P->K.rp[n]);
        double nq = 0, nu = 0;
        for (int64_t e = 0; e < n; ++e) nq += std::norm(q[e]), nu += std::norm(u[e]);
        const double al = std::abs(lam[i]);
        cres[c] = std::sqrt(nq) / ((op.P->nK + al * op.P->nC + al * al * op.P->nM) * std::sqrt(nu));
        if (!(cres[c] <= tol)) all = false;
        for (auto& z : u) z /= std::sqrt(nu);
        cvec[c] = std::move(u);
      }
    }
    out.lam.clear();
    out.res = cres;
    for (int c = 0; c < nev; ++c) out.lam.push_back(lam[ord[c]]);
    out.vec = cvec;
    std::vector<int> sel(mm, 0);
    bool deflate = false;
    if (all) {
      std::vector<double> d;
      for (int c = 0; c < nev; ++c) d.push_back(std::abs(lam[ord[c]] - sig));
      std::sort(d.begin(), d.end());
      bool improved = prev.empty();
      for (size_t i = 0; i < d.size() && !improved; ++i)
        if (d[i] < prev[i] * (1 - 1e-8)) improved = true;
      if (!guard_on || !improved || gp >= 64) {
        out.ok = true;
        break;
      }
      prev = d;
      ++gp;
      pass_cycles = 0;
      deflate = true;
      for (int c = 0; c < nev; ++c) sel[ord[c]] = 1;
    } else {
      for (int c = 0; c < std::min(keep_t, m - bs); ++c) sel[ord[c]] = 1;
    }
    int p = 0;
    for (int v : sel) p += v;
    std::vector<int> s2 = sel;
    schur_move_front(T, Z, s2);
    // V <- V Z[:, :p]; H <- [T_p; b^T]
#pragma omp parallel for schedule(dynamic, 1)
    for (int c = 0; c < p; ++c) {
      std::fill(V2[c].begin(), V2[c].end(), cd{});
      for (int t = 0; t < mm; ++t) k_axpy(Z(t, c), V[t].data(), V2[c].data(), n2);
    }
    if (L) L->add(RST, static_cast<double>(mm) * p * n2);
    // new residual rows E Z_p (E = H(mm.., m0..mm); bs = 1: beta Z(m-1, :))
    std::vector<cd> EZ(static_cast<size_t>(bs) * p, 0.0);
    for (int a = 0; a < bs; ++a)
      for (int c = 0; c < p; ++c)
        for (int q = 0; q < bs; ++q) EZ[a + static_cast<size_t>(c) * bs] += H(mm + a, m0 + q) * Z(m0 + q, c);
    H = DM(m + bs);
    for (int c = 0; c < p; ++c)
      for (int i = 0; i <= c; ++i) H(i, c) = T(i, c);
    for (int c = 0; c < p; ++c) V[c].swap(V2[c]);
    if (deflate) {
      fresh(seed + 0x1000003ull * gp, p);
    } else {
      for (int a = 0; a < bs; ++a)
        for (int c = 0; c < p; ++c) H(p + a, c) = EZ[a + static_cast<size_t>(c) * bs];
      for (int a = 0; a < bs; ++a) V[p + a] = V[mm + a];
    }
    k = p;
  }
  out.cycles = cycles;
  out.guard = gp;
  out.nconv = 0;
  for (double x : out.res) out.nconv += x <= tol;
  return out;
}

// Per-category timing of Arnoldi steps j0 .. j0+nsteps-1 (SURVEY.md §8(d)
// d4: the CPU path's per-cycle split). The basis is filled with seeded
// uniform vectors: the work per step (operator application, two CGS passes
// over j+1 vectors with their B-products, B-norm) equals a real step's, only
// the values differ. out[0..3] = ms in {SpMV, triangular solves, CGS2
// dot/axpy, other vector work}.
void step_profile(Operator& op, int j0, int nsteps, uint64_t seed, double* out) {
  using clk = std::chrono::steady_clock;
  auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const int64_t n = op.n, n2 = 2 * n;
  std::vector<std::vector<cd>> V(j0 + nsteps + 1, std::vector<cd>(n2));
  uint64_t st = seed;
  for (auto& v : V)
    for (auto& x : v) x = uni(st);
  std::vector<cd> r(n2), w(n2), t1(n), t2(n);
  double tsp = 0, tso = 0, tcg = 0, tot = 0;
  for (int j = j0; j < j0 + nsteps; ++j) {
    const cd* v = V[j].data();
    auto a = clk::now();
    spmv(op.P->C, v, t1.data(), nullptr);
    spmv(op.P->M, v, t2.data(), nullptr);
    auto b = clk::now();
    axpy(op.s, t2.data(), t1.data(), n, nullptr);
    auto c = clk::now();
    spmv(op.P->M, v + n, t2.data(), nullptr);
    auto d = clk::now();
    axpy(1.0, t2.data(), t1.data(), n, nullptr);
    auto e = clk::now();
    solve_factored(*op.F, t1.data(), r.data(), nullptr);
    auto f = clk::now();
    k_scal(-1.0, r.data(), n);
    for (int64_t i = 0; i < n; ++i) r[n + i] = v[i];
    axpy(op.s, r.data(), r.data() + n, n, nullptr);
    auto g = clk::now();
    tsp += ms(a, b) + ms(c, d);
    tot += ms(b, c) + ms(d, e) + ms(f, g);
    tso += ms(e, f);
    std::vector<cd> h(j + 1);
    for (int pass = 0; pass < 2; ++pass) {
      a = clk::now();
      op.bvec(r.data(), w.data(), nullptr);
      b = clk::now();
      dots(V, j + 1, w.data(), n2, h.data(), nullptr);
      axpys(V, j + 1, h.data(), r.data(), n2, -1.0, nullptr);
      c = clk::now();
      tsp += ms(a, b);
      tcg += ms(b, c);
    }
    a = clk::now();
    op.bvec(r.data(), w.data(), nullptr);
    b = clk::now();
    const double beta = std::sqrt(std::max(0.0, k_dotc(r.data(), w.data(), n2).real()));
    for (int64_t i = 0; i < n2; ++i) V[j + 1][i] = r[i] / beta;
    c = clk::now();
    tsp += ms(a, b);
    tcg += ms(b, c);
  }
  out[0] = tsp, out[1] = tso, out[2] = tcg, out[3] = tot;
}

// scale_pencil: varsigma = sqrt(maxabs K /
// maxabs M); the scaled pencil is (K, varsigma C,
// varsigma^2 M), whose eigenvalues are gamma = lambda / varsigma. Zero M -> errc 6.
double scale_pencil(Pencil& P) {
  double mk = 0, mm = 0;
  for (const cd& v : P.K.val) mk = std::max(mk, std::abs(v));
  for (const cd& v : P.M.val) mm = std::max(mm, std::abs(v));
  if (!(mm > 0)) throw OracleError{6, "scale_pencil: zero M norm"};
  const double s = std::sqrt(mk / mm), s2 = s * s;
  for (cd& v : P.C.val) v *= s;
  for (cd& v : P.M.val) v *= s2;
  return s;
}

// solve_generalized_hermitian (Alg. 1, Remark 3):
// A u = lambda B u, A Hermitian, B HPD, real shift s. The reference path's
// restatement: the oracle's complex multifrontal LU of A - s B, S = (A - s
// B)^{-1} B, the three-term Lanczos recurrence (alpha_j = v_j^H B S v_j,
// beta_j = ||r||_B) with a full CGS2 reorthogonalisation pass per step whose
// coefficients are not added to T (selective reorthogonalisation always
// engaged), thick restart keeping the p Ritz vectors nearest the shift (T =
// diag(theta) bordered by beta_m y_m), cyclic-Jacobi eigenvalues of the real
// symmetric T, explicit residuals ||A u - lambda B u|| / ((||A||_1 + |lambda|
// ||B||_1) ||u||).
void jacobi_sym(std::vector<double> A, int n, std::vector<double>& w, std::vector<double>& Z) {
  Z.assign(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i) Z[i + static_cast<size_t>(i) * n] = 1.0;
  auto a = [&](int i, int j) -> double& { return A[i + static_cast<size_t>(j) * n]; };
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) tot += a(i, j) * a(i, j), off += i != j ? a(i, j) * a(i, j) : 0.0;
    if (off <= 1e-30 * tot) break;
    for (int p = 0; p + 1 < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (a(p, q) == 0.0) continue;
        const double th = (a(q, q) - a(p, p)) / (2.0 * a(p, q));
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), sn = t * c;
        for (int k = 0; k < n; ++k) {
          const double x = a(k, p), y = a(k, q);
          a(k, p) = c * x - sn * y, a(k, q) = sn * x + c * y;
        }
        for (int k = 0; k < n; ++k) {
          const double x = a(p, k), y = a(q, k);
          a(p, k) = c * x - sn * y, a(q, k) = sn * x + c * y;
        }
        for (int k = 0; k < n; ++k) {
          double& x = Z[k + static_cast<size_t>(p) * n];
          double& y = Z[k + static_cast<size_t>(q) * n];
          const double zx = x, zy = y;
          x = c * zx - sn * zy, y = sn * zx + c * zy;
        }
      }
  }
  w.resize(n);
  for (int i = 0; i < n; ++i) w[i] = a(i, i);
}

struct GhOut {
  std::vector<double> lam, res;
  int cycles = 0;
  bool ok = false;
};

GhOut solve_generalized_hermitian(const Csr& A, const Csr& B, const Factor& F, double s, int nev, int m, double tol,
                                  uint64_t seed, int max_restarts) {
  const int64_t n = A.n;
  const int keep = nev + std::min(20, m - nev - 1);
  std::vector<std::vector<cd>> V(m + 1, std::vector<cd>(n));
  std::vector<cd> r(n), w(n), t(n);
  auto bvec = [&](const cd* x, cd* y) { spmv(B, x, y, nullptr); };
  auto apply = [&](const cd* v, cd* out) {
    bvec(v, t.data());
    solve_factored(F, t.data(), out, nullptr);
  };
  const double nA = norm1(A), nB = norm1(B);
  {
    uint64_t st = seed;
    for (int64_t i = 0; i < n; ++i) r[i] = uni(st);
    bvec(r.data(), w.data());
    const double b = std::sqrt(k_dotc(r.data(), w.data(), n).real());
    for (int64_t i = 0; i < n; ++i) V[0][i] = r[i] / b;
  }
  std::vector<double> T(static_cast<size_t>(m + 1) * (m + 1), 0.0), beta(m + 1, 0.0);
  auto Tc = [&](int i, int j) -> double& { return T[i + static_cast<size_t>(j) * (m + 1)]; };
  int k = 0;
  GhOut out;
  while (out.cycles < max_restarts) {
    ++out.cycles;
    int mm = m;
    for (int j = k; j < m; ++j) {
      apply(V[j].data(), r.data());
      double alpha = 0.0;
      for (int pass = 0; pass < 2; ++pass) {
        bvec(r.data(), w.data());
        std::vector<cd> h(j + 1);
        dots(V, j + 1, w.data(), n, h.data(), nullptr);
        axpys(V, j + 1, h.data(), r.data(), n, -1.0, nullptr);
        alpha += h[j].real();
      }
      bvec(r.data(), w.data());
      beta[j] = std::sqrt(std::max(0.0, k_dotc(r.data(), w.data(), n).real()));
      Tc(j, j) = alpha;
      Tc(j + 1, j) = Tc(j, j + 1) = beta[j];
      for (int64_t i = 0; i < n; ++i) V[j + 1][i] = r[i] / beta[j];
      if (beta[j] <= 1e-14 * std::max(1.0, std::fabs(alpha))) {
        mm = j + 1;
        break;
      }
    }
    std::vector<double> Tm(static_cast<size_t>(mm) * mm), th, Y;
    for (int j = 0; j < mm; ++j)
      for (int i = 0; i < mm; ++i) Tm[i + static_cast<size_t>(j) * mm] = Tc(i, j);
    jacobi_sym(Tm, mm, th, Y);
    std::vector<int> ord(mm);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(),
                     [&](int a_, int b_) { return std::fabs(1.0 / th[a_]) < std::fabs(1.0 / th[b_]); });
    const double bm = mm < m ? 0.0 : beta[m - 1];
    const int nw = std::min(nev, mm);
    bool all = true;
    for (int c = 0; c < nw; ++c)
      if (!(std::fabs(bm * Y[(mm - 1) + static_cast<size_t>(ord[c]) * mm]) / std::fabs(th[ord[c]]) <= 1e3 * tol))
        all = false;
    if (all || mm < m) {
      out.lam.clear();
      out.res.clear();
      all = true;
      for (int c = 0; c < nw; ++c) {
        const int i = ord[c];
        std::vector<cd> x(n, 0.0), y(mm);
        for (int q = 0; q < mm; ++q) y[q] = Y[q + static_cast<size_t>(i) * mm];
        axpys(V, mm, y.data(), x.data(), n, 1.0, nullptr);
        const double lam = s + 1.0 / th[i];
        std::vector<cd> ax(n), bx(n);
        spmv(A, x.data(), ax.data(), nullptr);
        spmv(B, x.data(), bx.data(), nullptr);
        double rr = 0, xx = 0;
        for (int64_t e = 0; e < n; ++e) rr += std::norm(ax[e] - lam * bx[e]), xx += std::norm(x[e]);
        const double res = std::sqrt(rr) / ((nA + std::fabs(lam) * nB) * std::sqrt(xx));
        out.lam.push_back(lam);
        out.res.push_back(res);
        if (!(res <= tol)) all = false;
      }
      if (all || mm < m) {
        out.ok = all;
        break;
      }
    }
    // thick restart
    const int p = std::min(keep, m - 1);
    std::vector<std::vector<cd>> V2(p + 1, std::vector<cd>(n, 0.0));
    for (int c = 0; c < p; ++c)
      for (int q = 0; q < mm; ++q) k_axpy(Y[q + static_cast<size_t>(ord[c]) * mm], V[q].data(), V2[c].data(), n);
    V2[p] = V[mm];
    for (int c = 0; c <= p; ++c) V[c].swap(V2[c]);
    std::fill(T.begin(), T.end(), 0.0);
    for (int c = 0; c < p; ++c) {
      Tc(c, c) = th[ord[c]];
      Tc(p, c) = Tc(c, p) = bm * Y[(mm - 1) + static_cast<size_t>(ord[c]) * mm];
    }
    k = p;
  }
  return out;
}

}  // namespace oracle

// ============================================================================
// C-ABI for tests (ctypes). Complex arrays are interleaved (re, im) doubles.
// ============================================================================
namespace {
thread_local std::string g_err;
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const oracle::OracleError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
oracle::Csr make_csr(int64_t n, const int64_t* rp, const int32_t* col, const double* val_c) {
  oracle::Csr A;
  A.n = n;
  A.rp.assign(rp, rp + n + 1);
  A.col.assign(col, col + rp[n]);
  A.val.resize(rp[n]);
  for (int64_t k = 0; k < rp[n]; ++k) A.val[k] = cd(val_c[2 * k], val_c[2 * k + 1]);
  return A;
}
struct OracleFactor {
  std::shared_ptr<oracle::Symbolic> S;
  oracle::Csr A;
  oracle::Factor F;
};
struct OracleEig {
  std::shared_ptr<oracle::Symbolic> S;
  oracle::Pencil P;  // the (possibly scaled) pencil the Krylov iteration sees
  double varsigma = 1.0;
  oracle::Csr Q;
  oracle::Factor F;
  oracle::Ledger L;
  std::unique_ptr<oracle::Operator> op;
  double t_factor_ms = 0;
};
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

// Host threads of the oracle's factorization (OpenMP; <= 0: all cores).
// Results are bit-identical for every thread count.
void oracle_set_threads(int n) { omp_set_num_threads(n > 0 ? n : omp_get_num_procs()); }
int oracle_get_threads() { return omp_get_max_threads(); }

int oracle_kind() {
#ifdef ORACLE_REF_KERN
  return 1;
#else
  return 0;
#endif
}

// Symbolic analysis: permutation + front sizes (graph derivation)
int oracle_symbolic(int64_t n, const int64_t* rp, const int32_t* col, const int32_t* box, int elems,
                    int leaf, int32_t* perm, int32_t* nfronts, int32_t* npiv, int32_t* nf, int32_t* parent,
                    int64_t* struct_nnz_l) {
  return guarded([&] {
    const oracle::Symbolic S = oracle::symbolic(n, rp, col, box, elems, leaf);
    std::copy(S.perm.begin(), S.perm.end(), perm);
    *nfronts = static_cast<int32_t>(S.node_rows.size());
    for (size_t f = 0; f < S.node_rows.size(); ++f) {
      if (npiv) npiv[f] = S.node_npiv[f];
      if (nf) nf[f] = static_cast<int32_t>(S.node_rows[f].size());
      if (parent) parent[f] = S.node_parent[f];
    }
    if (struct_nnz_l) *struct_nnz_l = S.struct_nnz_l;
  });
}

int oracle_factor_create(int64_t n, const int64_t* rp, const int32_t* col, const double* val_c,
                         const int32_t* box, int elems, int leaf, void** out, int64_t* swaps,
                         double* fa_macs) {
  return guarded([&] {
    auto h = std::make_unique<OracleFactor>();
    h->A = make_csr(n, rp, col, val_c);
    h->S = std::make_shared<oracle::Symbolic>(oracle::symbolic(n, rp, col, box, elems, leaf));
    h->F = oracle::lu_factorize(*h->S, h->A, nullptr);
    if (swaps) *swaps = h->F.swaps;
    if (fa_macs) *fa_macs = h->F.fa_macs;
    *out = h.release();
  });
}

// Symbolic analysis kept as a handle, so a timed numeric factorization
// (bench.py --impl reference) excludes the ordering / elimination tree.
int oracle_symbolic_create(int64_t n, const int64_t* rp, const int32_t* col, const int32_t* box, int elems,
                           int leaf, void** out) {
  return guarded([&] {
    *out = new std::shared_ptr<oracle::Symbolic>(
        std::make_shared<oracle::Symbolic>(oracle::symbolic(n, rp, col, box, elems, leaf)));
  });
}
void oracle_symbolic_destroy(void* s) { delete static_cast<std::shared_ptr<oracle::Symbolic>*>(s); }

// Numeric multifrontal LU of A on a symbolic handle (the values' pattern must
// be the one the symbolic analysis saw).
int oracle_factor_numeric(void* sym, int64_t n, const int64_t* rp, const int32_t* col, const double* val_c,
                          void** out, int64_t* swaps, double* fa_macs) {
  return guarded([&] {
    auto h = std::make_unique<OracleFactor>();
    h->S = *static_cast<std::shared_ptr<oracle::Symbolic>*>(sym);
    if (h->S->n != n) throw oracle::OracleError{7, "symbolic / matrix dimension mismatch"};
    h->A = make_csr(n, rp, col, val_c);
    h->F = oracle::lu_factorize(*h->S, h->A, nullptr);
    if (swaps) *swaps = h->F.swaps;
    if (fa_macs) *fa_macs = h->F.fa_macs;
    *out = h.release();
  });
}

int oracle_factor_solve(void* h, const double* b_c, double* x_c) {
  return guarded([&] {
    auto* F = static_cast<OracleFactor*>(h);
    oracle::solve_factored(F->F, reinterpret_cast<const cd*>(b_c), reinterpret_cast<cd*>(x_c), nullptr);
  });
}

// Front f (postorder) as dense row-major nf x nf complex + ipiv.
int oracle_factor_front(void* h, int f, double* dense_c, int32_t* ipiv, int32_t* rows) {
  return guarded([&] {
    auto* F = static_cast<OracleFactor*>(h);
    const auto& Fr = F->F.fr.at(f);
    if (dense_c) {  // L\U (the consumed contribution block reads as zero)
      cd* D = reinterpret_cast<cd*>(dense_c);
      for (int i = 0; i < Fr.nf; ++i)
        for (int c = 0; c < Fr.nf; ++c)
          D[static_cast<size_t>(i) * Fr.nf + c] = (i < Fr.npiv || c < Fr.npiv) ? Fr.lu(i, c) : cd{};
    }
    if (ipiv) std::copy(Fr.ipiv.begin(), Fr.ipiv.end(), ipiv);
    if (rows) std::copy(Fr.rows.begin(), Fr.rows.end(), rows);
  });
}

void oracle_factor_destroy(void* h) { delete static_cast<OracleFactor*>(h); }

// Quadratic eigensolve. K, C, M real or complex interleaved; sigma real.
// Quadratic eigensolve. K, C, M real or complex interleaved; sigma real.
// sym: an oracle_symbolic_create handle (NULL: analyse here from box/elems).
int oracle_eig_create2(void* sym, int64_t n, const int64_t* rp, const int32_t* col, const double* K_c,
                       const double* C_c, const double* M_c, const int32_t* box, int elems, int leaf,
                       double sigma, int scaling, void** out) {
  return guarded([&] {
    auto h = std::make_unique<OracleEig>();
    h->P.K = make_csr(n, rp, col, K_c);
    h->P.C = make_csr(n, rp, col, C_c);
    h->P.M = make_csr(n, rp, col, M_c);
    if (scaling) h->varsigma = oracle::scale_pencil(h->P);
    const double s = sigma / h->varsigma;  // the shift in the scaled variable gamma
    h->P.nK = oracle::norm1(h->P.K);
    h->P.nC = oracle::norm1(h->P.C);
    h->P.nM = oracle::norm1(h->P.M);
    h->Q = h->P.K;
    for (size_t k = 0; k < h->Q.val.size(); ++k)
      h->Q.val[k] = h->P.K.val[k] + s * h->P.C.val[k] + s * s * h->P.M.val[k];
    if (sym) {
      h->S = *static_cast<std::shared_ptr<oracle::Symbolic>*>(sym);
      if (h->S->n != n) throw oracle::OracleError{7, "symbolic / pencil dimension mismatch"};
    } else {
      h->S = std::make_shared<oracle::Symbolic>(oracle::symbolic(n, rp, col, box, elems, leaf));
    }
    const auto t0 = std::chrono::steady_clock::now();
    h->F = oracle::lu_factorize(*h->S, h->Q, &h->L);
    h->t_factor_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    h->op = std::make_unique<oracle::Operator>();
    h->op->P = &h->P;
    h->op->F = &h->F;
    h->op->s = s;
    h->op->n = n;
    *out = h.release();
  });
}

int oracle_eig_create(int64_t n, const int64_t* rp, const int32_t* col, const double* K_c, const double* C_c,
                      const double* M_c, const int32_t* box, int elems, int leaf, double sigma, void** out) {
  return oracle_eig_create2(nullptr, n, rp, col, K_c, C_c, M_c, box, elems, leaf, sigma, 0, out);
}

// scale_pencil on its own: C, M (complex interleaved) scaled in place.
int oracle_scale_pencil(int64_t n, const int64_t* rp, const int32_t* col, const double* K_c, double* C_c,
                        double* M_c, double* varsigma) {
  return guarded([&] {
    oracle::Pencil P;
    P.K = make_csr(n, rp, col, K_c);
    P.C = make_csr(n, rp, col, C_c);
    P.M = make_csr(n, rp, col, M_c);
    *varsigma = oracle::scale_pencil(P);
    std::memcpy(C_c, P.C.val.data(), sizeof(cd) * P.C.val.size());
    std::memcpy(M_c, P.M.val.data(), sizeof(cd) * P.M.val.size());
  });
}

double oracle_eig_varsigma(void* h) { return static_cast<OracleEig*>(h)->varsigma; }

// Front sizes of a symbolic handle (postorder): npiv, nf (either may be NULL).
int oracle_symbolic_fronts(void* sym, int32_t* nfronts, int32_t* npiv, int32_t* nf) {
  return guarded([&] {
    const oracle::Symbolic& S = **static_cast<std::shared_ptr<oracle::Symbolic>*>(sym);
    *nfronts = static_cast<int32_t>(S.node_rows.size());
    for (size_t f = 0; f < S.node_rows.size(); ++f) {
      if (npiv) npiv[f] = S.node_npiv[f];
      if (nf) nf[f] = static_cast<int32_t>(S.node_rows[f].size());
    }
  });
}

double oracle_eig_factor_ms(void* h) { return static_cast<OracleEig*>(h)->t_factor_ms; }

int oracle_eig_apply(void* h, const double* v_c, double* r_c) {
  return guarded([&] {
    auto* E = static_cast<OracleEig*>(h);
    E->op->apply(reinterpret_cast<const cd*>(v_c), reinterpret_cast<cd*>(r_c), &E->L);
  });
}

// b_inner: x_u^H y_u + x_l^H M y_l (one B-product, one dot)
int oracle_eig_b_inner(void* h, const double* x_c, const double* y_c, double* out_c) {
  return guarded([&] {
    auto* E = static_cast<OracleEig*>(h);
    const int64_t n2 = 2 * E->op->n;
    std::vector<cd> w(n2);
    E->op->bvec(reinterpret_cast<const cd*>(y_c), w.data(), &E->L);
    const cd r = oracle::dot(reinterpret_cast<const cd*>(x_c), w.data(), n2, &E->L);
    out_c[0] = r.real();
    out_c[1] = r.imag();
  });
}

// arnoldi_run: V (m+1) x 2n row-major, H (m+1) x m column-major (complex).
int oracle_eig_arnoldi(void* h, const double* v1_c, int m, double* V_c, double* H_c) {
  return guarded([&] {
    auto* E = static_cast<OracleEig*>(h);
    std::vector<std::vector<cd>> V;
    oracle::DM H(m + 1);
    oracle::arnoldi_run(*E->op, reinterpret_cast<const cd*>(v1_c), m, V, H, &E->L);
    const int64_t n2 = 2 * E->op->n;
    if (V_c)
      for (int j = 0; j <= m; ++j) std::memcpy(V_c + 2 * j * n2, V[j].data(), sizeof(cd) * n2);
    if (H_c)
      for (int j = 0; j < m; ++j)
        for (int i = 0; i <= m; ++i) {
          H_c[2 * (i + j * (m + 1))] = H(i, j).real();
          H_c[2 * (i + j * (m + 1)) + 1] = H(i, j).imag();
        }
  });
}

// CostLedger counters (sparse.hpp:57-103): {ops, macs} x {fa, fb, mv, vv, check, restart}
void oracle_eig_ledger(void* h, double* out) {
  const auto* E = static_cast<OracleEig*>(h);
  for (int c = 0; c < 6; ++c) out[2 * c] = static_cast<double>(E->L.ops[c]), out[2 * c + 1] = E->L.macs[c];
}
void oracle_eig_ledger_reset(void* h) { static_cast<OracleEig*>(h)->L = oracle::Ledger{}; }

int oracle_eig_solve_quadratic_block(void* h, int nev, int m, double tol, uint64_t seed, int max_restarts,
                                     int guard, int block, int min_steps, double* lam_c, double* res, double* vec_c,
                                     int32_t* stats, double* ledger) {
  return guarded([&] {
    auto* E = static_cast<OracleEig*>(h);
    const int bs = std::max(1, block);
    const int mk = m > 0 ? m : 2 * nev + 1;
    if (bs > 1 && (mk < nev + bs || mk + bs > 2 * E->op->n)) throw oracle::OracleError{2, "oracle: m too small for the block"};
    const oracle::EigOut o = oracle::solve_quadratic(*E->op, nev, mk, tol, seed, max_restarts, guard, &E->L, bs,
                                                     min_steps > 0 ? min_steps : 1);
    for (int i = 0; i < nev && i < static_cast<int>(o.lam.size()); ++i) {
      lam_c[2 * i] = o.lam[i].real() * E->varsigma;  // lambda = varsigma gamma
      lam_c[2 * i + 1] = o.lam[i].imag() * E->varsigma;
      res[i] = o.res[i];
      if (vec_c && !o.vec[i].empty())
        std::memcpy(vec_c + 2 * i * E->op->n, o.vec[i].data(), sizeof(cd) * E->op->n);
    }
    if (stats) stats[0] = o.cycles, stats[1] = o.guard, stats[2] = o.nconv, stats[3] = o.ok;
    if (ledger)
      for (int c = 0; c < 6; ++c) ledger[2 * c] = static_cast<double>(E->L.ops[c]), ledger[2 * c + 1] = E->L.macs[c];
    if (!o.ok) throw oracle::OracleError{4, "oracle: not converged within max_restarts"};
  });
}

int oracle_eig_solve_quadratic(void* h, int nev, int m, double tol, uint64_t seed, int max_restarts,
                               int guard, double* lam_c, double* res, double* vec_c, int32_t* stats,
                               double* ledger) {
  return oracle_eig_solve_quadratic_block(h, nev, m, tol, seed, max_restarts, guard, 1, 1, lam_c, res, vec_c, stats,
                                          ledger);
}

void oracle_eig_destroy(void* h) { delete static_cast<OracleEig*>(h); }

// solve_generalized_hermitian: real A, B (values, not
// interleaved) on one pattern; lam / res: double[nev] (nearest the shift first);
// stats: {cycles, ok}.
int oracle_gh_solve(int64_t n, const int64_t* rp, const int32_t* col, const double* a, const double* b,
                    const int32_t* box, int elems, int leaf, double s, int nev, int m, double tol, uint64_t seed,
                    int max_restarts, double* lam, double* res, int32_t* stats) {
  return guarded([&] {
    std::vector<double> ac(2 * rp[n], 0.0), bc(2 * rp[n], 0.0), qc(2 * rp[n], 0.0);
    for (int64_t k = 0; k < rp[n]; ++k) ac[2 * k] = a[k], bc[2 * k] = b[k], qc[2 * k] = a[k] - s * b[k];
    const oracle::Csr A = make_csr(n, rp, col, ac.data()), B = make_csr(n, rp, col, bc.data()),
                      Q = make_csr(n, rp, col, qc.data());
    const oracle::Symbolic S = oracle::symbolic(n, rp, col, box, elems, leaf);
    const oracle::Factor F = oracle::lu_factorize(S, Q, nullptr);
    const int mk = m > 0 ? m : std::max(2 * nev, nev + 20);
    const oracle::GhOut o = oracle::solve_generalized_hermitian(A, B, F, s, nev, mk, tol, seed, max_restarts);
    for (int i = 0; i < nev && i < static_cast<int>(o.lam.size()); ++i) lam[i] = o.lam[i], res[i] = o.res[i];
    if (stats) stats[0] = o.cycles, stats[1] = o.ok;
    if (!o.ok) throw oracle::OracleError{4, "oracle: generalized Hermitian solve did not converge"};
  });
}

int oracle_eig_step_profile(void* h, int j0, int nsteps, uint64_t seed, double* out) {
  return guarded([&] { oracle::step_profile(*static_cast<OracleEig*>(h)->op, j0, nsteps, seed, out); });
}

// Raw kern:: entry points (for checking the restated kernels against the
// reference build and the product's SpMV).
void oracle_kern_spmv(int64_t n, const int64_t* rp, const int32_t* col, const double* val_c,
                      const double* x_c, double* y_c) {
  oracle::k_spmv(n, rp, col, reinterpret_cast<const cd*>(val_c), reinterpret_cast<const cd*>(x_c),
                 reinterpret_cast<cd*>(y_c));
}
void oracle_kern_dotc(const double* x_c, const double* y_c, int64_t n, double* out_c) {
  const cd r = oracle::k_dotc(reinterpret_cast<const cd*>(x_c), reinterpret_cast<const cd*>(y_c), n);
  out_c[0] = r.real();
  out_c[1] = r.imag();
}
uint64_t oracle_kern_elim(double* tile_c, int64_t ld, const double* lcol_c, const double* urow_c,
                          int64_t rows, int64_t cols) {
  return oracle::k_elim(reinterpret_cast<cd*>(tile_c), ld, reinterpret_cast<const cd*>(lcol_c),
                        reinterpret_cast<const cd*>(urow_c), rows, cols);
}

}  // extern "C"
