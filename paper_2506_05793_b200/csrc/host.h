// Private host-side declarations of libfastilu_b200 (not part of the ABI).
#pragma once
#include <cstdint>
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

}  // namespace fastilu
