// SPDX-License-Identifier: Apache-2.0
// Symbolic analysis: geometric nested dissection + multifrontal front
// structure (host C++, bit-exact integer work).
//
// nested_dissection_order as pinned in SURVEY.md
// App. B D1:
//   - recurse on element boxes, cutting the longer side (ties -> x) at
//     x0 + w/2;
//   - a DOF is in the separator iff its support straddles the cut
//     (first < mid <= last);
//   - order left subtree, right subtree, then the separator; ascending
//     original id inside a set;
//   - leaf when the node holds <= leaf DOFs or both box sides are < 2.
// One dense front per ND node: rows = node DOFs (pivots) followed by the
// ancestor-separator DOFs whose support overlaps the node's element box (the
// contribution block). The oracle derives the same fronts independently from
// the Liu elimination tree (oracle/symbolic_graph.cpp) and the tests require
// both to agree front by front.
#include <algorithm>
#include <functional>

#include "common.hpp"

namespace rqb {

namespace {

struct NDNode {
  int bx0, bx1, by0, by1;  // half-open element box
  std::vector<int32_t> piv;
  std::vector<int32_t> children;
};

struct NDBuilder {
  const int32_t* box;
  int leaf;
  std::vector<NDNode> nodes;

  int build(int bx0, int bx1, int by0, int by1, std::vector<int32_t>&& dofs) {
    const int w = bx1 - bx0, h = by1 - by0;
    NDNode node{bx0, bx1, by0, by1, {}, {}};
    if (static_cast<int>(dofs.size()) <= leaf || (w < 2 && h < 2)) {
      std::sort(dofs.begin(), dofs.end());
      node.piv = std::move(dofs);
      nodes.push_back(std::move(node));
      return static_cast<int>(nodes.size()) - 1;
    }
    const bool cutx = w >= h;
    const int mid = cutx ? bx0 + w / 2 : by0 + h / 2;
    std::vector<int32_t> sep, left, right;
    for (int32_t d : dofs) {
      const int first = cutx ? box[4 * d + 0] : box[4 * d + 2];
      const int last = cutx ? box[4 * d + 1] : box[4 * d + 3];
      if (first < mid && last >= mid)
        sep.push_back(d);
      else if (last < mid)
        left.push_back(d);
      else
        right.push_back(d);
    }
    dofs.clear();
    dofs.shrink_to_fit();
    std::vector<int32_t> kids;
    if (!left.empty()) {
      if (cutx)
        kids.push_back(build(bx0, mid, by0, by1, std::move(left)));
      else
        kids.push_back(build(bx0, bx1, by0, mid, std::move(left)));
    }
    if (!right.empty()) {
      if (cutx)
        kids.push_back(build(mid, bx1, by0, by1, std::move(right)));
      else
        kids.push_back(build(bx0, bx1, mid, by1, std::move(right)));
    }
    if (sep.empty() && kids.size() == 1) return kids[0];  // nothing to separate here
    std::sort(sep.begin(), sep.end());
    node.piv = std::move(sep);
    node.children = std::move(kids);
    nodes.push_back(std::move(node));
    return static_cast<int>(nodes.size()) - 1;
  }
};

inline bool overlaps(const int32_t* b, const NDNode& nd) {
  return b[0] <= nd.bx1 - 1 && b[1] >= nd.bx0 && b[2] <= nd.by1 - 1 && b[3] >= nd.by0;
}

}  // namespace

Symbolic nested_dissection(int64_t n, const int32_t* box, int elems, int leaf) {
  if (n <= 0) fail(errc::dimension, "empty system");
  if (leaf < 1) fail(errc::config, "leaf size must be positive");
  if (n > INT32_MAX / 2) fail(errc::dimension, "system too large for int32 indices");
  NDBuilder B{box, leaf, {}};
  std::vector<int32_t> all(n);
  for (int64_t i = 0; i < n; ++i) all[i] = static_cast<int32_t>(i);
  const int root = B.build(0, elems, 0, elems, std::move(all));
  if (root != static_cast<int>(B.nodes.size()) - 1) fail(errc::generic, "ND root is not last");

  Symbolic S;
  S.n = n;
  const int nf = static_cast<int>(B.nodes.size());
  S.fronts.resize(nf);
  S.perm.reserve(n);
  // Creation order is a postorder (children are built before their node).
  for (int f = 0; f < nf; ++f) {
    Front& F = S.fronts[f];
    F.start = static_cast<int32_t>(S.perm.size());
    F.npiv = static_cast<int32_t>(B.nodes[f].piv.size());
    for (int32_t d : B.nodes[f].piv) S.perm.push_back(d);
    F.children = B.nodes[f].children;
    for (int32_t c : F.children) S.fronts[c].parent = f;
  }
  if (static_cast<int64_t>(S.perm.size()) != n) fail(errc::generic, "ND lost DOFs");
  S.iperm.assign(n, -1);
  for (int64_t i = 0; i < n; ++i) S.iperm[S.perm[i]] = static_cast<int32_t>(i);

  // Contribution-block rows, top-down: CB(s) = {d in rows(parent) : support(d)
  // overlaps box(s)}, which equals the ancestor-separator DOFs overlapping s.
  std::vector<std::vector<int32_t>> rows(nf);  // new ids, pivots first
  for (int f = nf - 1; f >= 0; --f) {
    Front& F = S.fronts[f];
    std::vector<int32_t>& r = rows[f];
    r.reserve(F.npiv);
    for (int k = 0; k < F.npiv; ++k) r.push_back(F.start + k);
    if (F.parent >= 0) {
      for (int32_t g : rows[F.parent]) {
        const int32_t d = S.perm[g];
        if (overlaps(box + 4 * d, B.nodes[f])) r.push_back(g);
      }
    }
    F.nf = static_cast<int32_t>(r.size());
  }
  // Heights, offsets, statistics.
  int maxlev = 0;
  int64_t off = 0, rows_off = 0, cbo = 0;
  for (int f = 0; f < nf; ++f) {
    Front& F = S.fronts[f];
    int lev = 0;
    for (int32_t c : F.children) lev = std::max(lev, S.fronts[c].level + 1);
    F.level = lev;
    maxlev = std::max(maxlev, lev);
    F.ld = (F.nf + 3) & ~3;
    F.off = off;
    off += static_cast<int64_t>(F.ld) * F.nf;
    off = (off + 3) & ~int64_t(3);
    F.rows_off = rows_off;
    rows_off += F.nf;
    F.cbvec_off = cbo;
    const int64_t ncb = F.nf - F.npiv;
    cbo += ncb;
    const int64_t np = F.npiv, nff = F.nf;
    S.nnz_l += np * (np + 1) / 2 + np * ncb;
    S.nnz_u += np * (np + 1) / 2 + np * ncb;
    S.max_front = std::max<int64_t>(S.max_front, nff);
    S.max_npiv = std::max<int64_t>(S.max_npiv, np);
    for (int64_t k = 0; k < np; ++k) {
      const double r = static_cast<double>(nff - k - 1);
      S.flops_lu += r + 2.0 * r * r;
    }
    const double sch = 2.0 * np * static_cast<double>(ncb) * ncb;
    S.flops_schur += sch;
    if (nff >= 1024) S.flops_schur_large += sch;
  }
  S.pool = off;
  S.cbvec = cbo;
  S.rows.reserve(rows_off);
  double sum_nf = 0;
  for (int f = 0; f < nf; ++f) {
    S.rows.insert(S.rows.end(), rows[f].begin(), rows[f].end());
    sum_nf += S.fronts[f].nf;
  }
  S.level_fronts.assign(maxlev + 1, {});
  for (int f = 0; f < nf; ++f) S.level_fronts[S.fronts[f].level].push_back(f);
  S.trisolve_bytes = 8.0 * (S.nnz_l + S.nnz_u - n) + 4.0 * sum_nf + 32.0 * n;
  return S;
}

}  // namespace rqb
