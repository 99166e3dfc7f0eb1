// Private host-side declarations of libfastilu_b200 (not part of the ABI).
#pragma once
#include <cstdint>
#include <algorithm>
#include <vector>

namespace fastilu {

// Result of a symbolic ILU(k) over global rows [row0, row0 + rows()).
struct Pattern {
  int64_t row0 = 0;
  std::vector<int64_t> rp;    // rows()+1, rebased to 0
  std::vector<int32_t> ci;    // global columns, sorted per row
  std::vector<int8_t> lev;    // level of fill per entry
  int64_t rows() const { return rp.empty() ? 0 : (int64_t)rp.size() - 1; }
};

// Validation of CSR rows given with global index base g0 (row r of the arrays is global
// row g0 + r); columns must lie in [0, ncols).  Returns a fastilu_status value and the
// offending GLOBAL row in *bad.
int validate_csr(int64_t nrows, const int64_t *rp, const int32_t *ci, int64_t g0, int64_t ncols,
                 int nthreads, int64_t *bad);

// Half bandwidth max |i - j| over the given rows.
int64_t half_bandwidth(int64_t nrows, const int64_t *rp, const int32_t *ci, int64_t g0,
                       int nthreads);

// Symbolic ILU(K) (level of fill, sum rule) of the rows supplied (global rows
// [g0, g0 + nrows)), for output rows [o0, o1) (global, g0 <= o0 <= o1 <= g0 + nrows).
// Entries with column < g0 are ignored (outside the supplied window).  Rows are exact when
// every fill path of length <= K+1 starting at them stays inside [g0, ...): the caller
// guarantees o0 - g0 >= 2 (K+1) bandwidth or g0 == 0.  Parallel over row chunks, each
// recomputed from a private window that starts 2 (K+1) bandwidth rows below it.
int symbolic_iluk(int64_t nrows, const int64_t *rp, const int32_t *ci, int64_t g0, int64_t o0,
                  int64_t o1, int K, int nthreads, Pattern &out, int64_t *bad);

int hw_threads(int requested);

// Structure classes of the owned rows and their position programs (classes.cpp).
struct ClassProgram {
  std::vector<int32_t> row_class;   // per owned row
  std::vector<int64_t> class_off;   // nclasses + 1: byte offset of each class's program
  std::vector<int32_t> class_aoff;  // per class: offset of the A-position part
  std::vector<uint8_t> prog;        // positions in S_i (255 = absent)
  int64_t nclasses = 0, nuclasses = 0;
};

// rp/ci/dloc: local S structure (nloc rows, local columns); owned rows [r0, r1); arp/apos:
// A's row pointers (local rows) and the offset of each A entry inside its S row.  Returns
// false (no classes) if a row is longer than 254 entries or the caps are exceeded.
bool build_classes(const std::vector<int64_t> &rp, const std::vector<int32_t> &ci,
                   const std::vector<int32_t> &dloc, int64_t nloc, int64_t r0, int64_t r1,
                   const std::vector<int64_t> &arp, const std::vector<int32_t> &apos,
                   int nthreads, size_t max_bytes, int32_t max_classes, ClassProgram &out);

}  // namespace fastilu
