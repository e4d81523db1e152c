// SPDX-License-Identifier: Apache-2.0
// Host-side core types of the B200 build. Error categories mirror rq::errc
// (reference proj/include/rigaqep/types.hpp:14-23) so the C-ABI can return them
// unchanged.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace rqb {

enum class errc : int {
  generic = 1,
  config = 2,
  assembly = 3,
  solver = 4,
  verification = 5,
  domain = 6,
  dimension = 7,
  singular = 8,
};

class Error : public std::runtime_error {
 public:
  Error(errc code, const std::string& what) : std::runtime_error(what), code_(code) {}
  errc code() const noexcept { return code_; }

 private:
  errc code_;
};

[[noreturn]] inline void fail(errc code, const std::string& what) { throw Error(code, what); }

// ---------------------------------------------------------------------------
// Univariate spline space (own restatement of the reference bookkeeping,
// splines.hpp:24-64): uniform open knots on [0,1] with per-breakpoint
// multiplicities, element spans and basis support ranges.
struct Univariate {
  int degree = 1;
  int elems = 1;
  std::vector<int> mult;         // interior multiplicities, size elems-1
  std::vector<double> knots;
  std::vector<int> elem_span;    // knot-span index of element e
  std::vector<int> sup_first, sup_last;  // inclusive element support of basis i
  int nbasis() const { return static_cast<int>(knots.size()) - degree - 1; }
  int first_basis(int e) const { return elem_span[e] - degree; }
};

Univariate make_univariate(int degree, int elems, const std::vector<int>& mult);

enum class SpaceKind { curl = 0, div = 1 };

struct Tensor2 {
  Univariate sx, sy;
  int64_t nx() const { return sx.nbasis(); }
  int64_t ny() const { return sy.nbasis(); }
  int64_t dofs() const { return nx() * ny(); }
};

struct VectorSpace {
  SpaceKind kind = SpaceKind::div;
  int degree = 2, elems = 2, levels = 0;
  std::vector<int> separators;  // interior breakpoint indices (0-based)
  Tensor2 cx, cy;               // x-component, y-component
  int64_t Nx() const { return cx.dofs(); }
  int64_t N() const { return cx.dofs() + cy.dofs(); }
};

VectorSpace build_space(SpaceKind kind, int degree, int elems, int levels);
std::vector<int64_t> boundary_mask(const VectorSpace& vs);

// ---------------------------------------------------------------------------
// Real CSR pencil on one shared pattern (sparse.hpp:16-47 layout:
// int64 rowptr, int32 col).
struct Pencil {
  int64_t n_full = 0, n = 0;
  std::vector<int64_t> rowptr;
  std::vector<int32_t> col;
  std::vector<double> K, C, M;
  std::vector<int32_t> box;          // 4 per free DOF: x0 x1 y0 y1 (inclusive elements)
  std::vector<int64_t> free_to_full;
  int elems = 0;
};

// mask: constrained full DOF ids (sorted; default boundary_mask(vs));
// full_to_free_out: the free numbering used.
Pencil assemble_pencil(const VectorSpace& vs, double alpha, double beta, const std::vector<int64_t>* mask = nullptr,
                       std::vector<int64_t>* full_to_free_out = nullptr);
// The paper's vibroacoustic pencil: rigid
// edges constrained, absorbing edges (bit mask: left 1, right 2, bottom 4, top
// 8) carry the impedance terms alpha / beta.
Pencil assemble_acoustic(const VectorSpace& vs, double rho, double c, double alpha, double beta, int absorbing);
// The paper's conductive electromagnetic pencil: K = -(1/mu)
// curl-curl, M = eps mass, C = -i D with D the layer-weighted mass (sigma_x on
// the x-component, sigma_y on the y-component); P.C = 0, D returned.
struct EmLayer {
  double y0, y1, sx, sy;
};
Pencil assemble_em(const VectorSpace& vs, double mu, double eps, const std::vector<EmLayer>& layers,
                   std::vector<double>* D);

// Pieces shared by the host assembler and the device one (cuda/assembly.cu).
// Free numbering: full_to_free[g] = free id or -1 (constrained), free_to_full.
void free_numbering(const VectorSpace& vs, std::vector<int64_t>* full_to_free,
                    std::vector<int64_t>* free_to_full, const std::vector<int64_t>* mask = nullptr);
// Inclusive element support box {x0, x1, y0, y1} of every free DOF.
std::vector<int32_t> support_boxes(const VectorSpace& vs, const std::vector<int64_t>& free_to_full);

// Gauss tables of one direction of one component: values / first derivatives
// of the p+1 bases active on element e at point q ([e][q][a]), weights [e][q].
struct QuadTable {
  int p = 0, nq = 0;
  std::vector<double> val, der, wq;
  void build(const Univariate& u, const double* gx, const double* gw, int nq_);
  const double* v(int e, int q) const { return &val[(static_cast<size_t>(e) * nq + q) * (p + 1)]; }
  const double* d(int e, int q) const { return &der[(static_cast<size_t>(e) * nq + q) * (p + 1)]; }
  double w(int e, int q) const { return wq[static_cast<size_t>(e) * nq + q]; }
};
// (p+1)-point Gauss tables, tab[component][direction].
void quad_tables(const VectorSpace& vs, QuadTable tab[2][2]);
constexpr int kMaxAsmDegree = 12;

// Device assembly (f1): the same pencil, bit for bit, computed on the current
// CUDA device (pattern, element matrices, colour-ordered gather) and copied
// back. ms[0..5) (nullable): device ms of the pattern / element / gather
// stages, host ms of the O(n) preparation and of the copy back.
// keep (nullable): receives the device copies and K, C, M are then NOT copied
// back (P.K/C/M stay empty; the pattern is always copied).
struct DevicePencil;
Pencil assemble_pencil_device(const VectorSpace& vs, double alpha, double beta, double* ms,
                              DevicePencil* keep = nullptr);

// ---------------------------------------------------------------------------
// Symbolic multifrontal structure.
struct Front {
  int32_t parent = -1;
  int32_t npiv = 0, nf = 0;
  int32_t start = 0;      // first pivot (new index)
  int32_t level = 0;      // height batch
  int32_t ld = 0;         // leading dimension of the dense front
  int64_t off = 0;        // offset in the front pool (doubles)
  int64_t rows_off = 0;   // offset into Symbolic::rows
  int64_t cbvec_off = 0;  // offset of the forward-solve contribution vector
  std::vector<int32_t> children;
};

struct Symbolic {
  int64_t n = 0;
  std::vector<int32_t> perm, iperm;    // perm[new] = old
  std::vector<Front> fronts;           // postorder
  std::vector<int32_t> rows;           // concatenated front row lists (new ids)
  std::vector<std::vector<int32_t>> level_fronts;  // fronts per height batch
  int64_t pool = 0, cbvec = 0;
  int64_t nnz_l = 0, nnz_u = 0, max_front = 0, max_npiv = 0;
  double flops_lu = 0, flops_schur = 0, flops_schur_large = 0;
  double trisolve_bytes = 0;
};

Symbolic nested_dissection(int64_t n, const int32_t* box, int elems, int leaf);

// (The per-CSR-entry destination in the front pool — the scatter map — is
// built on the device: cuda/factor.cu scatter_map_k.)

// Threads of the host-side dense work (m x m Schur products, Ritz vectors):
// half the processors, at most 8 (the GPU-feeding thread and the driver's own
// threads keep the rest; spinning OpenMP workers on an oversubscribed host cost
// far more than they save).
int host_threads();

inline uint64_t splitmix64(uint64_t& x) {
  uint64_t z = (x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// uniform[-1,1) from the top 53 bits.
inline double splitmix_uniform(uint64_t& state) {
  return (static_cast<double>(splitmix64(state) >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
}

}  // namespace rqb
