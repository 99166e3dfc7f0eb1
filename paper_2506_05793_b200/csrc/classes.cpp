// Structure classes of the rows of S (host setup for the class-program sweep kernel).
//
// The sweep's index matching -- "where does u_kj of pivot k land in row i?" -- depends only on
// the relative structure of row i (column offsets j - i, A's entries inside S_i) and on the
// relative structure of the strict upper rows of its pivots.  Rows with identical structure
// share one small position map ("program"), computed once here instead of on every sweep:
//   prog[class] = for each pivot t of the class (ascending), for each entry e of U_k's strict
//                 upper row: the position of (i, k + off_e) inside S_i, or 255 if absent;
//                 then the position inside S_i of each entry of A_i.
// Stencil matrices have a few hundred classes (boundary layers), so the maps live in L1/L2 and
// the kernel reads one byte per candidate instead of a column index plus a search.  Matrices
// without such repetition exceed the size cap and use the hash-lookup kernel instead.
#include <atomic>
#include <cstring>
#include <thread>
#include <unordered_map>

#include "host.h"

namespace fastilu {

namespace {

uint64_t hash_vec(const int32_t *v, size_t n) {
  uint64_t h = 1469598103934665603ull ^ (uint64_t)n;
  for (size_t i = 0; i < n; i++) {
    h ^= (uint32_t)v[i];
    h *= 1099511628211ull;
    h ^= h >> 29;
  }
  return h;
}

// Dedup of signature vectors: id for each item, representatives kept for exact comparison.
struct Dedup {
  std::unordered_map<uint64_t, std::vector<std::pair<std::vector<int32_t>, int32_t>>> map;
  int32_t next = 0;
  // returns id, or -1 if the cap is exceeded
  int32_t id(const std::vector<int32_t> &sig, uint64_t h, int32_t cap) {
    auto &bucket = map[h];
    for (auto &e : bucket)
      if (e.first == sig) return e.second;
    if (next >= cap) return -1;
    bucket.emplace_back(sig, next);
    return next++;
  }
};

template <class F>
void par_rows(int64_t r0, int64_t r1, int T, F f) {
  std::vector<std::thread> th;
  for (int t = 0; t < T; t++)
    th.emplace_back([=]() { f(r0 + (r1 - r0) * t / T, r0 + (r1 - r0) * (t + 1) / T, t); });
  for (auto &x : th) x.join();
}

// Per-thread dedup, then a merge of the (few) thread-local representatives into global ids.
template <class SigF>
bool classify(int64_t r0, int64_t r1, int T, int32_t cap, SigF sigf, std::vector<int32_t> &ids,
              std::vector<int64_t> &reps) {
  ids.assign(r1 - r0, -1);
  std::vector<Dedup> loc(T);
  std::vector<std::vector<int64_t>> locrep(T);
  std::atomic<bool> over{false};
  par_rows(r0, r1, T, [&](int64_t a, int64_t b, int t) {
    std::vector<int32_t> sig;
    for (int64_t r = a; r < b && !over.load(std::memory_order_relaxed); r++) {
      sigf(r, sig);
      int32_t before = loc[t].next;
      int32_t i = loc[t].id(sig, hash_vec(sig.data(), sig.size()), cap);
      if (i < 0) {
        over = true;
        break;
      }
      if (loc[t].next != before) locrep[t].push_back(r);
      ids[r - r0] = i;
    }
  });
  if (over) return false;
  Dedup glob;
  std::vector<std::vector<int32_t>> remap(T);
  std::vector<int32_t> sig;
  reps.clear();
  for (int t = 0; t < T; t++) {
    for (int64_t r : locrep[t]) {
      sigf(r, sig);
      int32_t before = glob.next;
      int32_t g = glob.id(sig, hash_vec(sig.data(), sig.size()), cap);
      if (g < 0) return false;
      if (glob.next != before) reps.push_back(r);
      remap[t].push_back(g);
    }
  }
  par_rows(r0, r1, T, [&](int64_t a, int64_t b, int t) {
    for (int64_t r = a; r < b; r++) ids[r - r0] = remap[t][ids[r - r0]];
  });
  return true;
}

}  // namespace

bool build_classes(const std::vector<int64_t> &rp, const std::vector<int32_t> &ci,
                   const std::vector<int32_t> &dloc, int64_t nloc, int64_t r0, int64_t r1,
                   const std::vector<int64_t> &arp, const std::vector<int32_t> &apos,
                   int nthreads, size_t max_bytes, int32_t max_classes, ClassProgram &out) {
  out = ClassProgram();
  const int T = std::max(1, std::min<int>(nthreads, (int)(nloc / 8192 + 1)));
  for (int64_t r = r0; r < r1; r++)
    if (rp[r + 1] - rp[r] > 254) return false;  // positions are bytes, 255 = absent
  // 1) ids of the strict-upper structures (relative offsets) of every local row
  std::vector<int32_t> uid;
  std::vector<int64_t> urep;
  auto usig = [&](int64_t r, std::vector<int32_t> &s) {
    s.clear();
    for (int64_t p = rp[r] + dloc[r] + 1; p < rp[r + 1]; p++) s.push_back(ci[p] - (int32_t)r);
  };
  if (!classify(0, nloc, T, max_classes, usig, uid, urep)) return false;
  // 2) row classes of the owned rows: S_i offsets, A positions, pivots' U structures
  auto rsig = [&](int64_t r, std::vector<int32_t> &s) {
    s.clear();
    const int64_t b = rp[r], m = rp[r + 1] - b;
    s.push_back((int32_t)m);
    s.push_back(dloc[r]);
    s.push_back((int32_t)(arp[r + 1] - arp[r]));
    for (int64_t p = b; p < b + m; p++) s.push_back(ci[p] - (int32_t)r);
    for (int64_t q = arp[r]; q < arp[r + 1]; q++) s.push_back(apos[q]);
    for (int64_t p = b; p < b + dloc[r]; p++) s.push_back(uid[ci[p]]);
  };
  std::vector<int32_t> cls;
  std::vector<int64_t> reps;
  if (!classify(r0, r1, T, max_classes, rsig, cls, reps)) return false;
  // 3) one program per class, built from its representative row
  out.row_class = std::move(cls);
  out.class_off.resize(reps.size() + 1);
  out.class_aoff.resize(reps.size());
  size_t bytes = 0;
  for (size_t c = 0; c < reps.size(); c++) {
    const int64_t i = reps[c];
    out.class_off[c] = (int64_t)out.prog.size();
    const int64_t b = rp[i], e = rp[i + 1];
    for (int64_t t = b; t < b + dloc[i]; t++) {
      const int32_t k = ci[t];
      for (int64_t q = rp[k] + dloc[k] + 1; q < rp[k + 1]; q++) {
        const int32_t j = ci[q];
        const int32_t *f = std::lower_bound(ci.data() + t + 1, ci.data() + e, j);
        out.prog.push_back((f != ci.data() + e && *f == j) ? (uint8_t)(f - (ci.data() + b))
                                                           : (uint8_t)255);
      }
    }
    out.class_aoff[c] = (int32_t)(out.prog.size() - out.class_off[c]);
    for (int64_t q = arp[i]; q < arp[i + 1]; q++) out.prog.push_back((uint8_t)apos[q]);
    bytes = out.prog.size();
    if (bytes > max_bytes) return false;
  }
  out.class_off[reps.size()] = (int64_t)out.prog.size();
  out.nclasses = (int64_t)reps.size();
  out.nuclasses = (int64_t)urep.size();
  return true;
}

}  // namespace fastilu
