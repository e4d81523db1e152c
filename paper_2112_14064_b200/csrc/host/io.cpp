// SPDX-License-Identifier: Apache-2.0
// Wire formats: Matrix Market exchange files for the
// pencil matrices and for dense vectors, and the eigenpair JSON dump.
//
// Same files as the reference's writers (sparse.cpp:121-174:
// write_matrix_market / read_matrix_market / write_matrix_market_vector;
// SPEC.md:269, 371, 503): "coordinate real|complex general" with 1-based
// indices in CSR order, 17 significant digits ("%.17g" == ostream precision
// 17), complex entries as "re im" pairs; reading sums duplicate entries and
// returns sorted CSR (from_triplets, sparse.cpp:99-118). The eigenpair dump is
// the JSON array of {re, im, residual} of SPEC.md:503.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>
#include <string>

#include "common.hpp"
#include "io.hpp"

namespace rqb {

namespace {

struct File {
  FILE* f = nullptr;
  File(const std::string& path, const char* mode) : f(std::fopen(path.c_str(), mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

// ostream << double at precision 17 (default float field) == "%.17g"
inline int put_double(char* p, double v) { return std::snprintf(p, 32, "%.17g", v); }

}  // namespace

void write_mm_csr(int64_t n, const int64_t* rowptr, const int32_t* col, const double* re, const double* im,
                  const std::string& path) {
  File out(path, "wb");
  if (!out.f) fail(errc::generic, "cannot open '" + path + "' for writing");
  const int64_t nnz = rowptr[n];
  bool real = true;
  if (im)
    for (int64_t k = 0; k < nnz && real; ++k) real = im[k] == 0.0;
  std::fprintf(out.f, "%%%%MatrixMarket matrix coordinate %s general\n", real ? "real" : "complex");
  std::fprintf(out.f, "%lld %lld %lld\n", static_cast<long long>(n), static_cast<long long>(n),
               static_cast<long long>(nnz));
  std::string buf;
  buf.reserve(1 << 20);
  char line[128];
  for (int64_t r = 0; r < n; ++r)
    for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) {
      int len = std::snprintf(line, sizeof(line), "%lld %d ", static_cast<long long>(r + 1), col[k] + 1);
      len += put_double(line + len, re[k]);
      if (!real) {
        line[len++] = ' ';
        len += put_double(line + len, im[k]);
      }
      line[len++] = '\n';
      buf.append(line, len);
      if (buf.size() > (1u << 20) - 128) {
        if (std::fwrite(buf.data(), 1, buf.size(), out.f) != buf.size())
          fail(errc::generic, "write failed for '" + path + "'");
        buf.clear();
      }
    }
  if (std::fwrite(buf.data(), 1, buf.size(), out.f) != buf.size() || std::fflush(out.f) != 0)
    fail(errc::generic, "write failed for '" + path + "'");
}

void write_mm_vector(int64_t n, const double* re, const double* im, const std::string& path) {
  File out(path, "wb");
  if (!out.f) fail(errc::generic, "cannot open '" + path + "' for writing");
  std::fprintf(out.f, "%%%%MatrixMarket matrix array complex general\n%lld 1\n", static_cast<long long>(n));
  char line[96];
  for (int64_t i = 0; i < n; ++i) {
    int len = put_double(line, re[i]);
    line[len++] = ' ';
    len += put_double(line + len, im ? im[i] : 0.0);
    line[len++] = '\n';
    if (std::fwrite(line, 1, len, out.f) != static_cast<size_t>(len))
      fail(errc::generic, "write failed for '" + path + "'");
  }
  if (std::fflush(out.f) != 0) fail(errc::generic, "write failed for '" + path + "'");
}

CsrFile read_mm_csr(const std::string& path) {
  std::ifstream is(path);
  if (!is) fail(errc::generic, "cannot open '" + path + "'");
  std::string line;
  if (!std::getline(is, line) || line.rfind("%%MatrixMarket", 0) != 0)
    fail(errc::generic, "not a Matrix Market file: " + path);
  const bool complex_vals = line.find("complex") != std::string::npos;
  if (line.find("pattern") != std::string::npos) fail(errc::generic, "pattern matrices not supported: " + path);
  if (line.find("coordinate") == std::string::npos) fail(errc::generic, "not a coordinate matrix: " + path);
  while (std::getline(is, line))
    if (!line.empty() && line[0] != '%') break;
  long long rows = 0, cols = 0, nnz = 0;
  {
    std::istringstream hs(line);
    hs >> rows >> cols >> nnz;
    if (!hs || rows != cols || rows < 0 || nnz < 0) fail(errc::generic, "bad Matrix Market header in " + path);
  }
  struct T {
    int32_t r, c;
    double re, im;
  };
  std::vector<T> t(static_cast<size_t>(nnz));
  for (long long k = 0; k < nnz; ++k) {
    long long r, c;
    double vr, vi = 0.0;
    is >> r >> c >> vr;
    if (complex_vals) is >> vi;
    if (!is) fail(errc::generic, "truncated Matrix Market body in " + path);
    if (r < 1 || r > rows || c < 1 || c > cols) fail(errc::generic, "index out of range in " + path);
    t[k] = {static_cast<int32_t>(r - 1), static_cast<int32_t>(c - 1), vr, vi};
  }
  // from_triplets: sorted by (row, column), duplicates summed (file order)
  std::stable_sort(t.begin(), t.end(), [](const T& a, const T& b) { return a.r != b.r ? a.r < b.r : a.c < b.c; });
  CsrFile m;
  m.n = rows;
  m.complex_values = complex_vals;
  m.rowptr.assign(rows + 1, 0);
  for (size_t k = 0; k < t.size();) {
    size_t e = k;
    double sr = 0.0, si = 0.0;
    while (e < t.size() && t[e].r == t[k].r && t[e].c == t[k].c) {
      sr += t[e].re;
      si += t[e].im;
      ++e;
    }
    m.col.push_back(t[k].c);
    m.re.push_back(sr);
    m.im.push_back(si);
    ++m.rowptr[t[k].r + 1];
    k = e;
  }
  for (long long i = 0; i < rows; ++i) m.rowptr[i + 1] += m.rowptr[i];
  return m;
}

std::string eigenpairs_json(int n, const double* re, const double* im, const double* res) {
  std::string s = "[";
  char num[32];
  for (int i = 0; i < n; ++i) {
    s += i ? ",\n  {\"re\": " : "\n  {\"re\": ";
    put_double(num, re[i]);
    s += num;
    s += ", \"im\": ";
    put_double(num, im[i]);
    s += num;
    s += ", \"residual\": ";
    put_double(num, res[i]);
    s += num;
    s += "}";
  }
  s += n ? "\n]" : "]";
  return s;
}

}  // namespace rqb
