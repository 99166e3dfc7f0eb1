// Host-side block structure for the block sweep (bsr.cu): detection of block-dense ILU(k)
// patterns and the per-target pivot-block lists.  Target block (I,J) receives, for every pivot
// block K of block row I with K < min(I,J) and (K,J) in S, the BS scalar terms k = BS K + c
// (c ascending); listing K ascending reproduces the scalar sweep's ascending-k order
// (reading R2).
#include "blocks.h"

#include <algorithm>
#include <atomic>
#include <thread>

namespace fastilu {

static bool is_block_dense(const std::vector<int64_t> &rp, const std::vector<int32_t> &ci,
                           int64_t n, int bs, int nthreads) {
  if (n <= 0 || n % bs) return false;
  const int64_t nb = n / bs;
  std::atomic<bool> ok{true};
  const int T = std::max(1, std::min<int>(nthreads, (int)(nb / 2048 + 1)));
  std::vector<std::thread> th;
  for (int t = 0; t < T; t++)
    th.emplace_back([&, t]() {
      const int64_t a = nb * t / T, e = nb * (t + 1) / T;
      for (int64_t I = a; I < e && ok.load(std::memory_order_relaxed); I++) {
        const int64_t r0 = bs * I, p0 = rp[r0], m = rp[r0 + 1] - p0;
        if (m % bs) { ok = false; break; }
        for (int64_t q = 0; q < m; q += bs) {
          const int32_t c0 = ci[p0 + q];
          if (c0 % bs) { ok = false; break; }
          for (int c = 1; c < bs; c++)
            if (ci[p0 + q + c] != c0 + c) { ok = false; break; }
        }
        for (int d = 1; d < bs && ok; d++) {
          const int64_t pd = rp[r0 + d];
          if (rp[r0 + d + 1] - pd != m) { ok = false; break; }
          for (int64_t q = 0; q < m; q++)
            if (ci[pd + q] != ci[p0 + q]) { ok = false; break; }
        }
      }
    });
  for (auto &x : th) x.join();
  return ok;
}

bool build_blocks(const std::vector<int64_t> &rp, const std::vector<int32_t> &ci, int64_t n,
                  int nthreads, int64_t max_terms, BlockPattern &bp) {
  int bs = 0;
  for (int cand : {4, 3, 2})
    if (is_block_dense(rp, ci, n, cand, nthreads)) {
      bs = cand;
      break;
    }
  if (!bs) return false;
  const int64_t nb = n / bs;
  BlockPattern B;
  B.bs = bs;
  B.nb = nb;
  B.bptr.resize(nb + 1);
  for (int64_t I = 0; I <= nb; I++) B.bptr[I] = rp[bs * I] / (bs * bs);
  B.nblk = B.bptr[nb];
  if (B.nblk >= (int64_t)INT32_MAX) return false;
  B.brow.resize(B.nblk);
  B.bcol.resize(B.nblk);
  B.bdiag.assign(nb, -1);
  for (int64_t I = 0; I < nb; I++) {
    const int64_t p0 = rp[bs * I];
    for (int64_t b = B.bptr[I]; b < B.bptr[I + 1]; b++) {
      const int32_t J = ci[p0 + bs * (b - B.bptr[I])] / bs;
      B.brow[b] = (int32_t)I;
      B.bcol[b] = J;
      if (J == I) B.bdiag[I] = (int32_t)b;
    }
    if (B.bdiag[I] < 0) return false;
  }
  // term counts, then the lists (two passes over the same loops; per-thread marker arrays)
  const int T = std::max(1, std::min<int>(nthreads, (int)(nb / 1024 + 1)));
  B.tptr.assign(B.nblk + 1, 0);
  auto walk = [&](int t, bool fill) {
    std::vector<int32_t> mark(nb, -1);
    const int64_t a = nb * t / T, e = nb * (t + 1) / T;
    for (int64_t I = a; I < e; I++) {
      const int64_t b0 = B.bptr[I], b1 = B.bptr[I + 1];
      for (int64_t b = b0; b < b1; b++) mark[B.bcol[b]] = (int32_t)(b - b0);
      std::vector<int64_t> cur;
      if (fill) cur.assign(B.tptr.begin() + b0, B.tptr.begin() + b1);
      for (int64_t bk = b0; bk < B.bdiag[I]; bk++) {  // pivot blocks K < I, ascending
        const int32_t K = B.bcol[bk];
        for (int64_t u = B.bdiag[K] + 1; u < B.bptr[K + 1]; u++) {  // (K, J), J > K
          const int32_t q = mark[B.bcol[u]];
          if (q < 0) continue;
          if (fill) {
            int64_t &w = cur[q];
            B.terms[2 * w] = (int32_t)bk;
            B.terms[2 * w + 1] = (int32_t)u;
            w++;
          } else {
            B.tptr[b0 + q + 1]++;
          }
        }
      }
      for (int64_t b = b0; b < b1; b++) mark[B.bcol[b]] = -1;
    }
  };
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; t++) th.emplace_back(walk, t, false);
    for (auto &x : th) x.join();
  }
  for (int64_t b = 0; b < B.nblk; b++) B.tptr[b + 1] += B.tptr[b];
  B.nterms = B.tptr[B.nblk];
  if (B.nterms > max_terms) return false;
  B.terms.resize(2 * B.nterms);
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; t++) th.emplace_back(walk, t, true);
    for (auto &x : th) x.join();
  }
  bp = std::move(B);
  return true;
}

}  // namespace fastilu
