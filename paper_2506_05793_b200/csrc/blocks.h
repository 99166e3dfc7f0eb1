// Host-side block structure for the block (BSR) sweep (bsr.cu).  Private to libfastilu_b200.
#pragma once
#include <cstdint>
#include <vector>

namespace fastilu {

struct BlockPattern {
  int bs = 0;
  int64_t nb = 0, nblk = 0, nterms = 0;
  std::vector<int64_t> bptr;   // nb + 1
  std::vector<int32_t> brow;   // nblk
  std::vector<int32_t> bcol;   // nblk
  std::vector<int32_t> bdiag;  // nb
  std::vector<int64_t> tptr;   // nblk + 1
  std::vector<int32_t> terms;  // 2 nterms: (block (I,K), block (K,J)), K ascending
};

// Is the pattern S (rows [0, n), sorted columns, diagonal present) made of dense bs x bs blocks
// for some bs in {4, 3, 2}: rows bs I .. bs I + bs - 1 share one column list, made of whole
// aligned column groups?  If so, fill bp with the block pattern and every target block's pivot
// block pairs.  Returns false (bp untouched) if not block-dense or if the term list would exceed
// max_terms.
bool build_blocks(const std::vector<int64_t> &rp, const std::vector<int32_t> &ci, int64_t n,
                  int nthreads, int64_t max_terms, BlockPattern &bp);

}  // namespace fastilu
