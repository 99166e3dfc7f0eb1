// Host setup of libfastilu_b200: CSR validation and the symbolic ILU(k) pattern.
//
// Symbolic ILU(k) ("level-based ILU", PAPER.md:719 level of fill k; sum rule
// lev(i,j) = min(lev(i,j), lev(i,k) + lev(k,j) + 1) over pivots k < min(i,j); R7).
// Implementation: per row, a sorted singly linked list over the row's columns (Saad,
// "Iterative Methods for Sparse Linear Systems", Sec. 10.3.3 style).  The pivot cursor walks
// the list in ascending order; the strict upper row of each pivot is merged in behind a
// second cursor, inserting fill in place, so the list stays sorted and no sort is needed.
//
// Parallelism: the row-by-row recurrence only reaches back 2 (K+1) * bandwidth rows (a fill
// path of length <= K+1 moves at most (K+1) * bandwidth rows, and a U-row used by row i lies
// within (K+1) * bandwidth below it), so each chunk of rows is computed independently from a
// private window that starts that many rows below the chunk.  The chunks' rows are exact and
// are concatenated.
#include <algorithm>
#include <atomic>
#include <climits>
#include <cstring>
#include <thread>

#include "host.h"

namespace fastilu {

int hw_threads(int requested) {
  if (requested > 0) return requested;
  unsigned h = std::thread::hardware_concurrency();
  return h ? (int)h : 1;
}

template <class F>
static void parallel_for(int64_t n, int nthreads, F f) {
  if (nthreads <= 1 || n < 4096) {
    f(0, n, 0);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; t++) {
    int64_t a = n * t / nthreads, b = n * (t + 1) / nthreads;
    th.emplace_back([=]() { f(a, b, t); });
  }
  for (auto &x : th) x.join();
}

int validate_csr(int64_t nrows, const int64_t *rp, const int32_t *ci, int64_t g0, int64_t ncols,
                 int nthreads, int64_t *bad) {
  // status values mirror fastilu_status: 2 = BAD_MATRIX, 3 = MISSING_DIAG
  *bad = -1;
  if (rp[0] != 0) {
    *bad = g0;
    return 2;
  }
  std::atomic<int64_t> first_bad{INT64_MAX}, first_miss{INT64_MAX};
  parallel_for(nrows, nthreads, [&](int64_t a, int64_t b, int) {
    for (int64_t r = a; r < b; r++) {
      int64_t s = rp[r], e = rp[r + 1];
      int64_t g = g0 + r;
      bool ok = e >= s, diag = false;
      for (int64_t q = s; ok && q < e; q++) {
        int64_t j = ci[q];
        if (j < 0 || j >= ncols || (q > s && ci[q] <= ci[q - 1])) ok = false;
        if (j == g) diag = true;
      }
      if (!ok) {
        int64_t cur = first_bad.load();
        while (g < cur && !first_bad.compare_exchange_weak(cur, g)) {}
      } else if (!diag) {
        int64_t cur = first_miss.load();
        while (g < cur && !first_miss.compare_exchange_weak(cur, g)) {}
      }
    }
  });
  // report the first offending row in row order (a malformed row_ptr makes later rows moot)
  int64_t fb = first_bad.load(), fm = first_miss.load();
  if (fb == INT64_MAX && fm == INT64_MAX) return 0;
  if (fb <= fm) {
    *bad = fb;
    return 2;
  }
  *bad = fm;
  return 3;
}

int64_t half_bandwidth(int64_t nrows, const int64_t *rp, const int32_t *ci, int64_t g0,
                       int nthreads) {
  std::vector<int64_t> part(std::max(nthreads, 1), 0);
  parallel_for(nrows, nthreads, [&](int64_t a, int64_t b, int t) {
    int64_t m = 0;
    for (int64_t r = a; r < b; r++) {
      int64_t e = rp[r + 1], s = rp[r];
      if (e > s) {
        m = std::max<int64_t>(m, g0 + r - (int64_t)ci[s]);
        m = std::max<int64_t>(m, (int64_t)ci[e - 1] - (g0 + r));
      }
    }
    part[t] = m;
  });
  return *std::max_element(part.begin(), part.end());
}

// Window worker: rows [w0, o1) (global) of the supplied matrix, emits rows [c0, o1) into out.
static int window_symbolic(const int64_t *rp, const int32_t *ci, int64_t g0, int64_t w0,
                           int64_t c0, int64_t c1, int K, Pattern &out, int64_t *bad) {
  // column slots cover [w0, colmax]
  int64_t colmax = c1 - 1;
  for (int64_t g = w0; g < c1; g++) {
    int64_t r = g - g0;
    if (rp[r + 1] > rp[r]) colmax = std::max(colmax, (int64_t)ci[rp[r + 1] - 1]);
  }
  const int64_t width = colmax - w0 + 1;
  const int32_t END = -1;
  const int32_t UNSET = INT32_MAX;
  std::vector<int32_t> nxt(width, END), lev(width, UNSET);
  // window rows' patterns (needed as U-rows of later rows)
  std::vector<int64_t> wrp(c1 - w0 + 1, 0);
  std::vector<int32_t> wci;
  std::vector<int8_t> wlev;
  std::vector<int64_t> wdiag(c1 - w0, 0);
  wci.reserve((size_t)(rp[c1 - g0] - rp[w0 - g0]) * 2);
  wlev.reserve(wci.capacity());
  for (int64_t i = w0; i < c1; i++) {
    const int64_t r = i - g0;
    // list of slots (column - w0); head is a sentinel kept outside nxt
    int32_t head = END, tail = END;
    for (int64_t q = rp[r]; q < rp[r + 1]; q++) {
      int64_t j = ci[q];
      if (j < w0) continue;  // outside the window
      int32_t sl = (int32_t)(j - w0);
      lev[sl] = 0;
      nxt[sl] = END;
      if (tail == END) head = sl; else nxt[tail] = sl;
      tail = sl;
    }
    const int32_t islot = (int32_t)(i - w0);
    for (int32_t cur = head; cur != END && cur < islot; cur = nxt[cur]) {
      const int64_t krow = cur;  // pivot k = w0 + cur, its window row index
      const int32_t lk = lev[cur];
      int32_t ins = cur;  // insertion cursor: last list node with column < current j
      for (int64_t q = wdiag[krow] + 1; q < wrp[krow + 1]; q++) {
        const int32_t l = lk + (int32_t)wlev[q] + 1;
        if (l > K) continue;
        const int32_t js = (int32_t)(wci[q] - w0);
        while (nxt[ins] != END && nxt[ins] < js) ins = nxt[ins];
        if (nxt[ins] == js) {
          if (l < lev[js]) lev[js] = l;
        } else {
          nxt[js] = nxt[ins];
          nxt[ins] = js;
          lev[js] = l;
        }
        ins = js;
      }
    }
    const int64_t wr = i - w0;
    bool has_diag = false;
    for (int32_t cur = head; cur != END;) {
      if (cur == islot) {
        wdiag[wr] = (int64_t)wci.size();
        has_diag = true;
      }
      wci.push_back((int32_t)(cur + w0));
      wlev.push_back((int8_t)lev[cur]);
      lev[cur] = UNSET;
      int32_t nx = nxt[cur];
      nxt[cur] = END;
      cur = nx;
    }
    if (!has_diag) {
      *bad = i;
      return 3;
    }
    wrp[wr + 1] = (int64_t)wci.size();
  }
  // emit rows [c0, c1)
  const int64_t s0 = wrp[c0 - w0], s1 = wrp[c1 - w0];
  out.row0 = c0;
  out.rp.resize(c1 - c0 + 1);
  for (int64_t g = c0; g <= c1; g++) out.rp[g - c0] = wrp[g - w0] - s0;
  out.ci.assign(wci.begin() + s0, wci.begin() + s1);
  out.lev.assign(wlev.begin() + s0, wlev.begin() + s1);
  return 0;
}

int symbolic_iluk(int64_t nrows, const int64_t *rp, const int32_t *ci, int64_t g0, int64_t o0,
                  int64_t o1, int K, int nthreads, Pattern &out, int64_t *bad) {
  *bad = -1;
  out = Pattern();
  out.row0 = o0;
  if (o1 <= o0) {
    out.rp.assign(1, 0);
    return 0;
  }
  nthreads = hw_threads(nthreads);
  const int64_t bw = half_bandwidth(nrows, rp, ci, g0, nthreads);
  const int64_t margin = 2 * (int64_t)(K + 1) * std::max<int64_t>(bw, 1);
  const int64_t n = o1 - o0;
  // chunk count: enough chunks for the threads, each at least as long as the margin
  int64_t nchunks = std::min<int64_t>(nthreads, std::max<int64_t>(1, n / std::max<int64_t>(margin, 2048)));
  if (n < 65536) nchunks = 1;
  std::vector<Pattern> parts(nchunks);
  std::vector<int> st(nchunks, 0);
  std::vector<int64_t> bads(nchunks, -1);
  auto work = [&](int64_t c) {
    int64_t c0 = o0 + n * c / nchunks, c1 = o0 + n * (c + 1) / nchunks;
    int64_t w0 = (c == 0) ? std::max(g0, o0 - margin) : std::max(g0, c0 - margin);
    if (c == 0 && o0 - g0 <= margin) w0 = g0;
    st[c] = window_symbolic(rp, ci, g0, w0, c0, c1, K, parts[c], &bads[c]);
  };
  if (nchunks == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (int64_t c = 0; c < nchunks; c++) th.emplace_back(work, c);
    for (auto &t : th) t.join();
  }
  for (int64_t c = 0; c < nchunks; c++)
    if (st[c]) {
      *bad = bads[c];
      return st[c];
    }
  // concatenate
  std::vector<int64_t> off(nchunks + 1, 0);
  for (int64_t c = 0; c < nchunks; c++) off[c + 1] = off[c] + (int64_t)parts[c].ci.size();
  out.rp.resize(n + 1);
  out.ci.resize(off[nchunks]);
  out.lev.resize(off[nchunks]);
  auto cat = [&](int64_t c) {
    const Pattern &p = parts[c];
    int64_t r0 = p.row0 - o0;
    for (int64_t r = 0; r < p.rows(); r++) out.rp[r0 + r] = p.rp[r] + off[c];
    if (!p.ci.empty()) {
      std::memcpy(out.ci.data() + off[c], p.ci.data(), p.ci.size() * sizeof(int32_t));
      std::memcpy(out.lev.data() + off[c], p.lev.data(), p.lev.size());
    }
  };
  if (nchunks == 1) {
    cat(0);
  } else {
    std::vector<std::thread> th;
    for (int64_t c = 0; c < nchunks; c++) th.emplace_back(cat, c);
    for (auto &t : th) t.join();
  }
  out.rp[n] = off[nchunks];
  return 0;
}

}  // namespace fastilu
