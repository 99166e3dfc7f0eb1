// Host-only dump of a generated sweep kernel, for compiling / inspecting it without a GPU:
//   g++ -O2 -std=c++17 -pthread -Ipaper_2506_05793_b200/csrc -Iinclude scripts/micro/gen_sweep.cpp \
//       paper_2506_05793_b200/csrc/{symbolic,tsell}.cpp -o /tmp/gen_sweep
//   /tmp/gen_sweep row|init|async K G THREADS PARTS > k.cu
//   nvcc -arch=sm_100a -cubin -Xptxas -v k.cu       (register / spill report)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "host.h"
#include "tsell.h"

using namespace fastilu;

int main(int argc, char **argv) {
  const char *mode = argc > 1 ? argv[1] : "row";
  const int K = argc > 2 ? atoi(argv[2]) : 1;
  const int g = argc > 3 ? atoi(argv[3]) : 40;
  const int threads = argc > 4 ? atoi(argv[4]) : 512;
  const int parts = argc > 5 ? atoi(argv[5]) : 4;
  // 27-point stencil, natural order, Dirichlet truncation
  std::vector<int64_t> rp{0};
  std::vector<int32_t> ci;
  for (int z = 0; z < g; z++)
    for (int y = 0; y < g; y++)
      for (int x = 0; x < g; x++) {
        for (int dz = -1; dz <= 1; dz++)
          for (int dy = -1; dy <= 1; dy++)
            for (int dx = -1; dx <= 1; dx++) {
              int X = x + dx, Y = y + dy, Z = z + dz;
              if (X < 0 || Y < 0 || Z < 0 || X >= g || Y >= g || Z >= g) continue;
              ci.push_back(X + g * (Y + g * Z));
            }
        rp.push_back((int64_t)ci.size());
      }
  const int64_t n = (int64_t)g * g * g;
  Pattern S;
  int64_t bad = -1;
  if (symbolic_iluk(n, rp.data(), ci.data(), 0, 0, n, K, 8, S, &bad)) return 1;
  Template T;
  std::vector<unsigned long long> mask;
  std::vector<int32_t> asrc;
  if (!build_template(S.rp, S.ci, n, rp, ci, 8, T, mask, asrc)) return 2;
  StagedCfg c{};
  std::string src;
  const unsigned opts = getenv("OPTS") ? (unsigned)atoi(getenv("OPTS"))
                                       : (kStagedFastDiv | kStagedOwnL | kStagedLastIssues);
  if (!strcmp(mode, "async"))
    src = sweep_source(T, threads, parts, 0, true, false, false, true);
  else if (!strcmp(mode, "init"))
    src = sweep_source_staged(T, threads, parts, 2, 0, true, &c, opts | kStagedFromAhat);
  else
    src = sweep_source_staged(T, threads, parts, 2, 0, false, &c, opts);
  fprintf(stderr, "W=%d c0=%d WA=%d terms=%zu rows=%d smem=%d box=32x%dx%d own=%d lds=%d tma=%lld\n", T.W, T.c0,
          T.WA, T.terms.size(), c.rows, c.smem, c.box_cols, c.box_slices, c.own_cols, c.lds_per_row,
          c.tma_bytes_per_tile);
  fputs(src.c_str(), stdout);
  return 0;
}
