// SPDX-License-Identifier: Apache-2.0
// Wire formats: Matrix Market files and the eigenpair JSON.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace rqb {

// CSR matrix read from a Matrix Market file (values split in re / im).
struct CsrFile {
  int64_t n = 0;
  bool complex_values = false;
  std::vector<int64_t> rowptr;
  std::vector<int32_t> col;
  std::vector<double> re, im;
};

// im may be nullptr (real matrix); a complex matrix whose imaginary parts are
// all zero is written as "real", like the reference's is_real() check
void write_mm_csr(int64_t n, const int64_t* rowptr, const int32_t* col, const double* re, const double* im,
                  const std::string& path);
void write_mm_vector(int64_t n, const double* re, const double* im, const std::string& path);
CsrFile read_mm_csr(const std::string& path);
std::string eigenpairs_json(int n, const double* re, const double* im, const double* res);

}  // namespace rqb
