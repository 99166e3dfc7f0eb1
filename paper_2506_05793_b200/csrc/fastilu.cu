// C ABI of libfastilu_b200 (include/fastilu.h): handle, host setup orchestration, device
// layouts, and the stream-ordered compute / apply sequences.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "../../include/fastilu.h"
#include "comm.h"
#include "device.h"
#include "host.h"
#include "blocks.h"
#include "jit.h"
#include "tsell.h"

#define FAIL(code)                                                                  \
  do {                                                                              \
    if (std::getenv("FASTILU_DEBUG"))                                               \
      fprintf(stderr, "fastilu: %s at %s:%d\n", #code, __FILE__, __LINE__);         \
    return code;                                                                    \
  } while (0)

using namespace fastilu;

struct fastilu_handle_s {
  int64_t err_index = -1;
  fastilu_options opt{};
  int K = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // fastilu_compute_host: value upload pipelined with the compute (copy stream, chunk events)
  cudaStream_t copy_stream = nullptr;
  cudaStream_t d2h_stream = nullptr;  // solve_host: x back per chunk during the upload
  std::vector<cudaEvent_t> chunk_ev;
  int chunk_b = 0;  // index of the event after the right-hand side's upload (solve_host)
  std::vector<cudaEvent_t> x_ev;  // solve_host pipeline: chunk c of x final
  std::vector<int64_t> h_arp;  // local A row pointers (offsets into the local values)
  double *d_r2c = nullptr;     // per-chunk residual sums (chunks x nsweeps)
  int r2c_cap = 0;
  // partition (global indices)
  int64_t n = 0, global_n = 0, row_begin = 0, n_lead = 0;
  int64_t G = 0, H = 0, lbase = 0, nloc = 0, E = 0;
  int64_t nnz_loc = 0, nnz_own = 0, own_off = 0;  // S entries (local rows), owned rows, offset
  int64_t nnzA_loc = 0, nnzA_own = 0;
  int64_t a_in_off = 0, a_in_nnz = 0;  // local A rows inside the caller's value array
  // host copies (owned rows) for introspection
  std::vector<int64_t> h_rp;
  std::vector<int32_t> h_ci;
  std::vector<int8_t> h_lev;
  // device structure
  int64_t *d_rp = nullptr;
  int32_t *d_ci = nullptr, *d_dloc = nullptr;
  int64_t *d_arp = nullptr;
  int32_t *d_aci = nullptr, *d_apos = nullptr, *d_adiag = nullptr;
  double *d_aval = nullptr;
  // device values
  double *d_vals[2] = {nullptr, nullptr}, *d_ud[2] = {nullptr, nullptr}, *d_ahat = nullptr;
  double *d_s = nullptr, *d_ad = nullptr;
  double *d_y = nullptr, *d_z[2] = {nullptr, nullptr}, *d_w[2] = {nullptr, nullptr};
  double *d_it = nullptr;  // solve_host pipeline: z^1..z^ntri, w^1..w^ntri
  double *d_vals3 = nullptr, *d_ud3 = nullptr;  // compute_host pipeline: third iterate buffer
  int it_cap = 0;
  double *d_bx = nullptr;  // apply_host staging (2 n)
  double *d_partials = nullptr, *d_r2 = nullptr;
  int hist_cap = 0;
  int32_t *d_rclass = nullptr, *d_caoff = nullptr;  // class-program sweep
  int64_t *d_coff = nullptr;
  uint8_t *d_prog = nullptr;
  int64_t nclasses = 0;
  // template-SELL fast path (tsell.h)
  bool tsell = false;
  Template T;
  int64_t nsl = 0;  // slices of 32 local rows
  int32_t *d_toff = nullptr, *d_toffA = nullptr, *d_tasrc = nullptr;
  int8_t *d_tw2a = nullptr;
  unsigned long long *d_tmask = nullptr;
  unsigned int *d_counter = nullptr;
  double *d_aT = nullptr;  // A's values in template slots (refreshed by set_values)
  // block path (bsr.cu, blocks.h): block-dense patterns, single GPU
  bool bsr = false;
  BsrDev B{};
  int64_t *d_bptr = nullptr, *d_tptr = nullptr;
  int32_t *d_brow = nullptr, *d_bcol = nullptr, *d_bdiag = nullptr;
  int2 *d_terms = nullptr;
  double *d_vb[2] = {nullptr, nullptr}, *d_ahb = nullptr;
  int bsr_grid = 0, bsr_threads = 256;
  size_t bsr_smem = 0;
  int bsr_minb = 1;
  int64_t bsr_nterms = 0;
  const double *vals_cur = nullptr, *ud_cur = nullptr;  // factors of the last compute
  std::vector<unsigned long long *> d_lmask;  // warm-up: presence masks of levels 0..K-1
  void *jit_sweep = nullptr;
  void *jit_sweep_first = nullptr;  // sweep 1 from iterate 0: A x A terms only
  void *jit_sweep_async = nullptr;  // the asynchronous kernel of the current block size
  std::vector<std::pair<int, void *>> jit_async;  // (parts, kernel), compiled on first use
  int async_ept = 0;                              // nonzeros per thread of the next async compute
  int async_parts = 0, async_rows = 0;
  // staged sweep (tsell.h StagedCfg): pivot rows through shared memory by TMA
  void *jit_st = nullptr, *jit_st_first = nullptr;
  void *jit_st_init = nullptr;  // sweep 1 with iterate 0 computed from ahat (single GPU)
  void *jit_scale = nullptr, *jit_ahat = nullptr;  // template-specialised a2 / a3 (tsell)
  void *jit_jac[2] = {nullptr, nullptr};            // template-specialised a8 / a9 sweeps
  void *jit_spmv = nullptr;                          // template-specialised y = A x (GMRES)
  StagedCfg st{}, st_init{};
  int st_grid = 0, st_init_grid = 0;
  int64_t st_ntiles = 0, st_init_ntiles = 0;
  struct alignas(64) TMapBuf {
    unsigned char b[128];
  } st_tmap[2], st_tmap_ahat;  // per iterate buffer d_vals[0/1]; over d_ahat
  TMapBuf st_tmap_own[2], st_tmap_own_ahat;  // own-row boxes (kStagedOwnL)
  TMapBuf st_tmap3, st_tmap_own3;  // over d_vals3
  int t_parts = 1, t_minb = 0, t_sstride = 1;
  bool t_prefetch = true;
  int t_threads = 128, t_grid = 1, t_regs = 0, t_spill = 0, t_rows_tile = 128;
  int64_t t_ntiles = 0;
  // GMRES workspace (allocated on first use)
  double *gm_V = nullptr, *gm_w = nullptr, *gm_ext = nullptr, *gm_u = nullptr, *gm_r = nullptr;
  double *gm_part = nullptr, *gm_c = nullptr, *gm_hbuf = nullptr;  // gm_hbuf pinned host
  int gm_reorth = 0;  // second Gram-Schmidt passes taken by the last fastilu_gmres
  int gm_retry = 0;   // DCGS2: explicit re-projections after a severe cancellation
  int gm_m = 0, G_spmv = 32;
  ErrFlags *d_err = nullptr;
  ErrFlags *h_err = nullptr;  // pinned
  double *h_r2 = nullptr;     // pinned, hist_cap
  // launch configuration
  SweepCfg scfg{};
  int G_init = 32, G_tri = 32;
  // state
  bool have_values = false, computed = false;
  int cur = 0;
  std::vector<double> resid;
  cudaEvent_t ev[6] = {};  // ev[5]: after sweep 1
  float t_sweep1 = 0.f;
  int last_ns = 0;
  float t_init = 0.f, t_sweeps = 0.f, t_apply = 0.f;
  bool apply_timed = false;  // ev[3] / ev[4] recorded by an apply
  Comm *comm = nullptr;
};

static const char *kStatus[] = {"FASTILU_OK",          "FASTILU_ERR_INVALID_ARG",
                                "FASTILU_ERR_BAD_MATRIX", "FASTILU_ERR_MISSING_DIAG",
                                "FASTILU_ERR_ZERO_DIAG", "FASTILU_ERR_ZERO_PIVOT",
                                "FASTILU_ERR_STATE",   "FASTILU_ERR_CUDA",
                                "FASTILU_ERR_NCCL",    "FASTILU_ERR_OOM",
                                "FASTILU_ERR_UNSUPPORTED"};

extern "C" const char *fastilu_status_string(fastilu_status s) {
  int i = (int)s;
  return (i >= 0 && i <= 10) ? kStatus[i] : "FASTILU_UNKNOWN";
}

extern "C" int64_t fastilu_error_index(fastilu_handle h) { return h ? h->err_index : -1; }

extern "C" void fastilu_default_options(fastilu_options *o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->omega = 1.0;
  o->omega_tri = 1.0;
  o->device = -1;
  o->stream = nullptr;
  o->num_threads = 0;
  o->rank = 0;
  o->nranks = 1;
  o->comm_kind = FASTILU_COMM_NONE;
  o->global_n = -1;
  o->row_begin = 0;
  o->n_lead = 0;
  o->shift = 0.0;
}

extern "C" int64_t fastilu_required_lead_rows(int64_t bandwidth, int level_k) {
  return 2 * (int64_t)(level_k + 1) * std::max<int64_t>(bandwidth, 1);
}

#define CU(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      if (std::getenv("FASTILU_DEBUG"))                                              \
        fprintf(stderr, "fastilu: %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, \
                __LINE__);                                                           \
      return e_ == cudaErrorMemoryAllocation ? FASTILU_ERR_OOM : FASTILU_ERR_CUDA;   \
    }                                                                                \
  } while (0)

template <class T>
static cudaError_t dalloc(T **p, int64_t count) {
  *p = nullptr;
  if (count <= 0) count = 1;
  return cudaMalloc((void **)p, sizeof(T) * (size_t)count);
}

// --------------------------------------------------------------------------- symbolic (host)
extern "C" fastilu_status fastilu_symbolic(int64_t n, const int64_t *row_ptr,
                                           const int32_t *col_idx, int level_k, int num_threads,
                                           int64_t *nnz_out, int64_t *row_ptr_out,
                                           int32_t *col_idx_out, int8_t *level_out,
                                           int64_t *bad_row) {
  if (bad_row) *bad_row = -1;
  if (n < 0 || !row_ptr || (n > 0 && !col_idx) || level_k < 0 || level_k > 127)
    FAIL(FASTILU_ERR_INVALID_ARG);
  int64_t bad = -1;
  int nt = hw_threads(num_threads);
  int st = validate_csr(n, row_ptr, col_idx, 0, n, nt, &bad);
  if (st) {
    if (bad_row) *bad_row = bad;
    return (fastilu_status)st;
  }
  Pattern pat;
  st = symbolic_iluk(n, row_ptr, col_idx, 0, 0, n, level_k, nt, pat, &bad);
  if (st) {
    if (bad_row) *bad_row = bad;
    return (fastilu_status)st;
  }
  if (nnz_out) *nnz_out = pat.rp[n];
  if (col_idx_out) {
    if (row_ptr_out) std::memcpy(row_ptr_out, pat.rp.data(), sizeof(int64_t) * (n + 1));
    std::memcpy(col_idx_out, pat.ci.data(), sizeof(int32_t) * pat.ci.size());
    if (level_out) std::memcpy(level_out, pat.lev.data(), pat.lev.size());
  }
  return FASTILU_OK;
}

extern "C" fastilu_status fastilu_symbolic_window(int64_t nrows, const int64_t *row_ptr,
                                                  const int32_t *col_idx, int64_t row0,
                                                  int64_t ncols, int64_t out_begin,
                                                  int64_t out_end, int level_k, int num_threads,
                                                  int64_t *nnz_out, int64_t *row_ptr_out,
                                                  int32_t *col_idx_out, int8_t *level_out,
                                                  int64_t *bad_row) {
  if (bad_row) *bad_row = -1;
  if (nrows < 0 || !row_ptr || (nrows > 0 && !col_idx) || level_k < 0 || level_k > 127 ||
      row0 < 0 || out_begin < row0 || out_end < out_begin || out_end > row0 + nrows ||
      ncols < row0 + nrows)
    FAIL(FASTILU_ERR_INVALID_ARG);
  int64_t bad = -1;
  int nt = hw_threads(num_threads);
  int st = validate_csr(nrows, row_ptr, col_idx, row0, ncols, nt, &bad);
  if (st) {
    if (bad_row) *bad_row = bad;
    return (fastilu_status)st;
  }
  Pattern pat;
  st = symbolic_iluk(nrows, row_ptr, col_idx, row0, out_begin, out_end, level_k, nt, pat, &bad);
  if (st) {
    if (bad_row) *bad_row = bad;
    return (fastilu_status)st;
  }
  const int64_t no = out_end - out_begin;
  if (nnz_out) *nnz_out = pat.rp[no];
  if (col_idx_out) {
    if (row_ptr_out) std::memcpy(row_ptr_out, pat.rp.data(), sizeof(int64_t) * (no + 1));
    std::memcpy(col_idx_out, pat.ci.data(), sizeof(int32_t) * pat.ci.size());
    if (level_out) std::memcpy(level_out, pat.lev.data(), pat.lev.size());
  }
  return FASTILU_OK;
}

// --------------------------------------------------------------------------- create
// Injective multiplicative hash of the column offsets j - i of every owned row:
// slot = ((uint32)(j - i) * mul) >> (32 - bits).  Returns false if none of the candidates works.
static bool find_offset_hash(const std::vector<int64_t> &rp, const std::vector<int32_t> &ci,
                             int64_t r0, int64_t r1, int64_t m_max, int nthreads, uint32_t *mul,
                             int *bits) {
  static const uint32_t kMul[] = {0x9E3779B1u, 0x85EBCA77u, 0xC2B2AE3Du, 0x27D4EB2Fu,
                                  0x165667B1u, 0xD3A2646Cu | 1u, 0xFD7046C5u, 0xB55A4F09u};
  if (m_max > 65535) return false;
  int b0 = 1;
  while ((1ll << b0) < 2 * std::max<int64_t>(m_max, 1)) b0++;
  for (int b = b0; b <= 12; b++) {
    for (uint32_t mu : kMul) {
      std::atomic<bool> bad{false};
      const int T = std::max(1, std::min<int>(nthreads, (int)((r1 - r0) / 4096 + 1)));
      std::vector<std::thread> th;
      for (int t = 0; t < T; t++)
        th.emplace_back([&, t]() {
          std::vector<int64_t> stamp((size_t)1 << b, -1);
          int64_t a = r0 + (r1 - r0) * t / T, e = r0 + (r1 - r0) * (t + 1) / T;
          for (int64_t r = a; r < e && !bad.load(std::memory_order_relaxed); r++) {
            for (int64_t p = rp[r]; p < rp[r + 1]; p++) {
              uint32_t h = ((uint32_t)(ci[p] - (int32_t)r) * mu) >> (32 - b);
              if (stamp[h] == r) {
                bad = true;
                break;
              }
              stamp[h] = r;
            }
          }
        });
      for (auto &x : th) x.join();
      if (!bad) {
        *mul = mu;
        *bits = b;
        return true;
      }
    }
  }
  return false;
}

static fastilu_status setup_configs(fastilu_handle h, const std::vector<int64_t> &rp,
                                    const std::vector<int32_t> &ci, int64_t m_max, double u_avg,
                                    double nl_avg, int64_t maxU, bool have_prog, int nthreads) {
  SweepCfg c{};
  int G = 4;
  while (G < u_avg && G < 32) G *= 2;
  c.G = G;
  c.threads = 512;
  c.cap_m = (int)std::max<int64_t>(4, (m_max + 3) / 4 * 4);
  c.E = (int)((std::max<int64_t>(maxU, 1) + G - 1) / G);
  if (c.E == 3) c.E = 4;
  c.prog = have_prog && c.E <= (G == 32 ? 4 : 2);
  if (c.prog) {
    const size_t gb = (((size_t)c.cap_m * 8 + (size_t)G * 24) + 15) & ~(size_t)15;
    while (c.threads > 64 && (size_t)(c.threads / G) * gb > 200 * 1024) c.threads /= 2;
    if ((size_t)(c.threads / G) * gb <= 220 * 1024) {
      c.smem = (size_t)(c.threads / G) * gb;
      int bps = 0;
      if (sweep_prog_configure(c, &bps) != cudaSuccess || bps < 1) return FASTILU_ERR_CUDA;
      const int sms = sm_count(h->device);
      const int64_t gpb = c.threads / G;
      const int64_t need = std::max<int64_t>(1, (h->n + gpb - 1) / gpb);
      c.grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * bps, need));
      c.chunk = gpb * 4;  // rows per block tile (4 rows per group)
      h->scfg = c;
      int gi = 4;
      while (gi < (double)h->nnz_own / std::max<int64_t>(h->n, 1) && gi < 32) gi *= 2;
      h->G_init = gi;
      int gt = 1;  // trisolve: 2 entries per lane in the fast path
      while (2 * gt < nl_avg && gt < 32) gt *= 2;
      h->G_tri = gt;
      return FASTILU_OK;
    }
    c.prog = false;
    c.threads = 512;
  }
  uint32_t mul = 0;
  int bits = 0;
  c.hash = find_offset_hash(rp, ci, h->G, h->G + h->n, m_max, nthreads, &mul, &bits);
  c.hmul = mul;
  c.hshift = c.hash ? 32 - bits : 0;
  c.hsize = c.hash ? (1 << bits) : 0;
  auto gbytes = [&](const SweepCfg &cc) {
    size_t b = (size_t)cc.cap_m * 12 + (size_t)cc.hsize * 2;
    return (b + 15) & ~(size_t)15;
  };
  while (c.threads > 32 && (size_t)(c.threads / G) * gbytes(c) > 200 * 1024) c.threads /= 2;
  if (c.threads < G || (size_t)(c.threads / G) * gbytes(c) > 220 * 1024)
    FAIL(FASTILU_ERR_UNSUPPORTED);  // a row of S too long for the shared-memory accumulator
  c.smem = (size_t)(c.threads / G) * gbytes(c);
  int bps = 0;
  if (sweep_configure(c, &bps) != cudaSuccess || bps < 1) return FASTILU_ERR_CUDA;
  const int sms = sm_count(h->device);
  const int64_t gpb = c.threads / G;
  const int64_t need = std::max<int64_t>(1, (h->n + gpb - 1) / gpb);
  c.grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * bps, need));
  c.chunk = gpb * 4;  // rows per block tile (4 rows per group)
  h->scfg = c;
  int gi = 4;
  while (gi < (double)h->nnz_own / std::max<int64_t>(h->n, 1) && gi < 32) gi *= 2;
  h->G_init = gi;
  int gt = 1;  // trisolve: 2 entries per lane in the fast path
  while (2 * gt < nl_avg && gt < 32) gt *= 2;
  h->G_tri = gt;
  return FASTILU_OK;
}

static TDev tdev(fastilu_handle h);

static fastilu_status upload_values(fastilu_handle h, const double *values, bool device) {
  cudaMemcpyKind kind = device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  CU(cudaMemcpyAsync(h->d_aval, values + h->a_in_off, sizeof(double) * h->nnzA_loc, kind,
                     h->stream));
  if (h->tsell) CU(launch_tsell_gather_a(tdev(h), h->d_aval, h->nloc, h->d_aT, h->stream));
  if (!device) CU(cudaStreamSynchronize(h->stream));
  h->have_values = true;
  h->computed = false;
  return FASTILU_OK;
}

// Template-SELL: compile the template-specialised sweep, allocate and upload the layout.
static fastilu_status setup_tsell(fastilu_handle h, const std::vector<unsigned long long> &mask,
                                  const std::vector<int32_t> &asrc) {
  const Template &T = h->T;
  h->nsl = (h->nloc + 31) / 32;
  const char *ev_th = std::getenv("FASTILU_TSELL_THREADS");
  const char *ev_pa = std::getenv("FASTILU_TSELL_PARTS");
  const char *ev_mb = std::getenv("FASTILU_TSELL_MINB");
  const int threads = ev_th ? std::max(32, atoi(ev_th) / 32 * 32) : 256;
  // targets split over 2 warps per row (measured best for W = 63 and 115, profiles/r1*)
  int parts = T.W > 16 ? 2 : 1;
  if (ev_pa) parts = std::max(1, atoi(ev_pa));
  // keep two 256-thread blocks per SM for templates whose accumulators fit 128 registers
  const int minb = ev_mb ? atoi(ev_mb) : (threads == 256 && T.W <= 72 ? 2 : 0);
  std::string log;
  // L2 prefetch of the next tile: measured slower at 256^3 (profiles/r1*), off by default
  const bool pf = std::getenv("FASTILU_TSELL_PREFETCH") &&
                  atoi(std::getenv("FASTILU_TSELL_PREFETCH")) != 0;
  h->t_prefetch = pf;
  const std::string src = sweep_source(T, threads, parts, minb, false, pf);
  if (jit_get(src, "fastilu_tsell_sweep", h->device, &h->jit_sweep, &log)) {
    if (std::getenv("FASTILU_DEBUG")) fprintf(stderr, "fastilu: JIT failed: %s\n", log.c_str());
    FAIL(FASTILU_ERR_UNSUPPORTED);
  }
  if (!std::getenv("FASTILU_NO_FIRST_SWEEP")) {
    const std::string s1 = sweep_source(T, threads, parts, minb, false, pf, true);
    if (jit_get(s1, "fastilu_tsell_sweep_first", h->device, &h->jit_sweep_first, &log))
      FAIL(FASTILU_ERR_UNSUPPORTED);
  }
  // staged sweep: default for templates with more than one pivot row per line of pivots
  // (27-pt ILU(k)); FASTILU_TSELL_STAGED=0/1 overrides
  {
    const char *ev = std::getenv("FASTILU_TSELL_STAGED");
    const bool want = ev ? atoi(ev) != 0 : T.W > 16;
    if (want) {
      const char *ev_st = std::getenv("FASTILU_TSELL_STAGES");
      const char *ev_sp = std::getenv("FASTILU_TSELL_ST_PARTS");
      const int nst = ev_st ? std::max(2, atoi(ev_st)) : 2;
      // ~32 targets per thread: 2 part-warps per slice for W = 63, 4 for W = 115
      const int sparts = ev_sp ? std::max(1, atoi(ev_sp)) : std::max(1, (T.W + 31) / 32);
      const char *ev_sth = std::getenv("FASTILU_TSELL_ST_THREADS");
      const char *ev_so = std::getenv("FASTILU_TSELL_ST_OPTS");
      const unsigned damp = h->opt.omega != 1.0 ? kStagedDamp : 0u;
      const unsigned base_opts = kStagedFastDiv | kStagedOwnL | kStagedLastIssues;
      // block shape and options of the full sweep, tried in order until one compiles and fits:
      //  - 2 part-warps per slice (W <= 64, 27-pt ILU(1)): 256-row tiles, one 512-thread block
      //    per SM, row-major boxes (c4 15.9 vs 16.8 ms for 3 sweeps against 128-row tiles;
      //    column-major boxes / no presence select measured neutral to 1 % slower,
      //    profiles/r2j_*);
      //  - 4 part-warps (27-pt ILU(2)): 160-row tiles, one 640-thread block (20 warps; 102
      //    registers fit because column-major boxes drop the per-pivot row-index split),
      //    column-major boxes without the presence selects: c3b full sweep 2.00 -> 1.57 ms
      //    (profiles/r2j_*); else 128-row tiles / 512 threads, row-major.
      // FASTILU_TSELL_ST_THREADS / _ST_OPTS override (one candidate).
      struct Cand { int threads; unsigned opts; };
      std::vector<Cand> cands;
      if (ev_sth || ev_so) {
        const int th = ev_sth ? std::max(32 * sparts, atoi(ev_sth) / (32 * sparts) * 32 * sparts)
                              : (sparts <= 2 ? 256 * sparts : 128 * sparts);
        cands.push_back({th, ev_so ? (unsigned)atoi(ev_so) : base_opts});
      } else {
        if (sparts >= 4)
          cands.push_back({160 * sparts, base_opts | kStagedColMajor | kStagedNoLSel});
        cands.push_back({sparts <= 2 ? 256 * sparts : 128 * sparts, base_opts});
      }
      const char *ev_smb = std::getenv("FASTILU_TSELL_ST_MINB");
      const int sminb = ev_smb ? atoi(ev_smb) : 0;
      StagedCfg c{};
      int sbps = 0, sthreads = 0;
      unsigned sopts = 0;
      bool ok_st = false;
      for (const auto &cd : cands) {
        sthreads = cd.threads;
        sopts = cd.opts | damp;
        c = StagedCfg{};
        const std::string s0 =
            sweep_source_staged(T, sthreads, sparts, nst, sminb, false, &c, sopts);
        const std::string s1 =
            sweep_source_staged(T, sthreads, sparts, nst, sminb, true, nullptr, sopts);
        if (std::getenv("FASTILU_DUMP_SRC")) fprintf(stderr, "%s\n", s0.c_str());
        sbps = 0;
        if (!jit_get(s0, "fastilu_tsell_sweep_st", h->device, &h->jit_st, &log) &&
            !jit_get(s1, "fastilu_tsell_sweep_st_first", h->device, &h->jit_st_first, &log) &&
            !jit_set_smem(h->jit_st, c.smem) && !jit_set_smem(h->jit_st_first, c.smem) &&
            !jit_occupancy(h->jit_st, c.threads, c.smem, &sbps) && sbps > 0) {
          int sregs = 0, sloc = 0, dummy = 0;
          jit_func_info(h->jit_st, &sregs, &sloc, c.threads, &dummy);
          if (sloc == 0 || &cd == &cands.back()) {  // a spilling candidate is not taken
            ok_st = true;
            break;
          }
        }
      }
      if (ok_st) {
        h->st = c;
        h->st_ntiles = std::max<int64_t>(1, (h->n + c.shift + c.rows - 1) / c.rows);
        // the first sweep with the init fused in
        StagedCfg ci{};
        // its stage (A's columns only) is small: FASTILU_TSELL_STAGES_INIT more ring slots
        const char *ev_si = std::getenv("FASTILU_TSELL_STAGES_INIT");
        const int nsi = ev_si ? std::max(2, atoi(ev_si)) : nst;
        // its own block shape (its A x A terms need half the full sweep's accumulators): for
        // 2-part templates (27-pt ILU(1)) one part-warp per slice and 384-row tiles (less box
        // overhang): c4 sweep 1 3.46 -> 2.93 ms; for 4-part templates (ILU(2)) two part-warps
        // and 256-row tiles: c3b 1.12 -> 0.84 ms (profiles/r1j_*, r1l_*).
        // FASTILU_TSELL_INIT_PARTS / _THREADS override.
        const char *ev_ip = std::getenv("FASTILU_TSELL_INIT_PARTS");
        const char *ev_it = std::getenv("FASTILU_TSELL_INIT_THREADS");
        const int iparts = ev_ip ? std::max(1, atoi(ev_ip))
                                 : (sparts == 2 ? 1 : sparts >= 4 ? 2 : sparts);
        const int ithreads =
            ev_it ? std::max(32 * iparts, atoi(ev_it) / (32 * iparts) * 32 * iparts)
            : ev_ip ? sthreads
            : sparts == 2 ? 384
            : sparts >= 4 ? 512
                          : sthreads;
        // column-major boxes for the init-fused sweep: c4 sweep 1 3.03 -> 2.94 ms, c3a 0.379
        // -> 0.368, c3b 0.838 -> 0.828 (profiles/r2j_*); FASTILU_TSELL_INIT_OPTS overrides
        const char *ev_io = std::getenv("FASTILU_TSELL_INIT_OPTS");
        const unsigned iopts =
            (ev_io ? (unsigned)atoi(ev_io)
                   : ev_so ? (unsigned)atoi(ev_so) : (base_opts | kStagedColMajor)) | damp;
        const std::string s2 = sweep_source_staged(T, ithreads, iparts, nsi, sminb, true, &ci,
                                                   iopts | kStagedFromAhat);
        int ibps = 0;
        if (!std::getenv("FASTILU_NO_FUSED_INIT") &&
            !jit_get(s2, "fastilu_tsell_sweep_st_init", h->device, &h->jit_st_init, &log) &&
            !jit_set_smem(h->jit_st_init, ci.smem) && ci.shift == c.shift &&
            !jit_occupancy(h->jit_st_init, ci.threads, ci.smem, &ibps) && ibps > 0) {
          h->st_init = ci;
          h->st_init_ntiles = std::max<int64_t>(1, (h->n + ci.shift + ci.rows - 1) / ci.rows);
          h->st_init_grid =
              (int)std::min<int64_t>((int64_t)sm_count(h->device) * ibps, h->st_init_ntiles);
        } else {
          h->jit_st_init = nullptr;
        }
        h->st_grid = (int)std::min<int64_t>((int64_t)sm_count(h->device) * sbps, h->st_ntiles);
        if (std::getenv("FASTILU_DEBUG")) {
          int sregs = 0, sloc = 0, dummy = 0;
          jit_func_info(h->jit_st, &sregs, &sloc, c.threads, &dummy);
          fprintf(stderr, "fastilu: staged threads=%d parts=%d rows=%d smem=%d regs=%d local=%d "
                  "blocks/SM=%d grid=%d\n", c.threads, c.parts, c.rows, c.smem, sregs, sloc, sbps,
                  h->st_grid);
        }
      } else {
        if (std::getenv("FASTILU_DEBUG"))
          fprintf(stderr, "fastilu: staged sweep unavailable: %s\n", log.c_str());
        h->jit_st = h->jit_st_first = nullptr;
      }
    }
  }
  // template-specialised scale / ahat kernels (FASTILU_NO_JIT_PREP=1 keeps the generic ones)
  if (!std::getenv("FASTILU_NO_JIT_PREP") && T.c0 >= 0 && T.w2a[T.c0] >= 0) {
    const std::string sp = prep_source(T, h->opt.nranks > 1);
    if (jit_get(sp, "fastilu_tsell_scale", h->device, &h->jit_scale, &log) ||
        jit_get(sp, "fastilu_tsell_ahat", h->device, &h->jit_ahat, &log))
      h->jit_scale = h->jit_ahat = nullptr;
  }
  // template-specialised streaming Jacobi sweeps (FASTILU_NO_JIT_JACOBI=1 keeps the generic)
  const char *ev_jm = std::getenv("FASTILU_JIT_JACOBI_MODE");
  const int jmode = ev_jm ? atoi(ev_jm) : 2;  // 2: interleaved (measured best: c4 apply 6.8 -> 5.8 ms; loads-first 11.0)
  if (!std::getenv("FASTILU_NO_JIT_JACOBI") && jmode > 0) {
    const std::string jl = jacobi_source(T, true, jmode == 1),
                      ju = jacobi_source(T, false, jmode == 1);
    if (jit_get(jl, "fastilu_tsell_jac_L", h->device, &h->jit_jac[0], &log) ||
        jit_get(ju, "fastilu_tsell_jac_U", h->device, &h->jit_jac[1], &log))
      h->jit_jac[0] = h->jit_jac[1] = nullptr;
  }
  // template-specialised SpMV for GMRES (FASTILU_NO_JIT_SPMV=1 keeps the CSR kernel): the 7-pt
  // config-5 matrix's CSR SpMV ran at ~2 TB/s (0.92 ms at 256^3, profiles/r2p_*)
  if (!std::getenv("FASTILU_NO_JIT_SPMV") && T.c0 >= 0) {
    if (jit_get(spmv_source(T), "fastilu_tsell_spmv", h->device, &h->jit_spmv, &log))
      h->jit_spmv = nullptr;
  }
  int bps = 0;
  jit_func_info(h->jit_sweep, &h->t_regs, &h->t_spill, threads, &bps);
  if (std::getenv("FASTILU_DEBUG"))
    fprintf(stderr, "fastilu: tsell W=%d c0=%d WA=%d terms=%zu regs=%d local=%d bps=%d\n", T.W,
            T.c0, T.WA, T.terms.size(), h->t_regs, h->t_spill, bps);
  if (bps < 1) FAIL(FASTILU_ERR_UNSUPPORTED);
  h->t_threads = threads;
  h->t_parts = parts;
  // slice stride of a tile: the template's grid line (smallest positive offset that is a
  // multiple of 32 rows), in slices; 1 if none
  // (measured neutral at 128^3/256^3 -- the sweep is not L1-bound -- so consecutive slices
  // stay the default; FASTILU_TSELL_SSTRIDE=g/32 enables it)
  h->t_sstride = 1;
  if (std::getenv("FASTILU_TSELL_SSTRIDE")) h->t_sstride = std::max(1, atoi(std::getenv("FASTILU_TSELL_SSTRIDE")));
  h->t_minb = minb;
  h->t_rows_tile = sweep_rows_per_tile(threads, parts);
  {
    const int64_t nsl_own = (h->n + 31) / 32, spt = h->t_rows_tile / 32, ss = h->t_sstride;
    h->t_ntiles = std::max<int64_t>(1, (nsl_own + spt * ss - 1) / (spt * ss) * ss);
  }
  h->t_grid = (int)std::min<int64_t>((int64_t)sm_count(h->device) * bps, h->t_ntiles);
  const int64_t nv = h->nsl * T.W * 32;
  for (int b = 0; b < 2; b++) {
    CU(dalloc(&h->d_vals[b], nv));
    CU(cudaMemset(h->d_vals[b], 0, sizeof(double) * nv));  // absent slots stay +0.0
  }
  CU(dalloc(&h->d_ahat, h->nsl * T.WA * 32));
  CU(cudaMemset(h->d_ahat, 0, sizeof(double) * h->nsl * T.WA * 32));
  CU(dalloc(&h->d_aT, h->nsl * T.WA * 32));
  CU(cudaMemset(h->d_aT, 0, sizeof(double) * h->nsl * T.WA * 32));
  CU(dalloc(&h->d_tmask, (int64_t)mask.size()));
  CU(dalloc(&h->d_tasrc, (int64_t)asrc.size()));
  CU(dalloc(&h->d_toff, T.W));
  CU(dalloc(&h->d_toffA, T.WA));
  CU(dalloc(&h->d_tw2a, T.W));
  CU(dalloc(&h->d_counter, 2));  // [1]: second launch of a split (halo-overlapped) sweep
  CU(dalloc(&h->d_partials,  // +2: a split sweep has one partial tile per launch more
            std::max<int64_t>(std::max(std::max(h->t_ntiles, h->st_ntiles), h->st_init_ntiles) + 2,
                              kSumsqBlocks)));
  // kStagedColMajor kernels take the swapped-dimension maps (box lands column-major)
  auto tmap = [](const StagedCfg &c, void *out, const double *base, int W, long long nsl,
                 int box_cols, int box_slices) {
    return c.colmajor ? jit_tmap_sell_cm(out, base, W, nsl, box_cols, box_slices)
                      : jit_tmap_sell(out, base, W, nsl, box_cols, box_slices);
  };
  if (h->jit_st)
    for (int b = 0; b < 2; b++)
      if (tmap(h->st, h->st_tmap[b].b, h->d_vals[b], T.W, h->nsl, h->st.box_cols,
               h->st.box_slices)) {
        if (std::getenv("FASTILU_DEBUG")) fprintf(stderr, "fastilu: tensor map failed\n");
        h->jit_st = h->jit_st_first = h->jit_st_init = nullptr;
      }
  if (h->jit_st_init && tmap(h->st_init, h->st_tmap_ahat.b, h->d_ahat, T.WA, h->nsl,
                             h->st_init.box_cols, h->st_init.box_slices))
    h->jit_st_init = nullptr;
  // own-row boxes: {32, own_cols, rows/32} (any valid map when the kernel does not use them)
  if (h->jit_st)
    for (int b = 0; b < 2; b++)
      if (tmap(h->st, h->st_tmap_own[b].b, h->d_vals[b], T.W, h->nsl,
               std::max(1, h->st.own_cols), h->st.rows / 32))
        h->jit_st = h->jit_st_first = h->jit_st_init = nullptr;
  if (h->jit_st_init && tmap(h->st_init, h->st_tmap_own_ahat.b, h->d_ahat, T.WA, h->nsl,
                             std::max(1, h->st_init.own_cols), h->st_init.rows / 32))
    h->jit_st_init = nullptr;
  CU(cudaMemset(h->d_counter, 0, 2 * sizeof(unsigned int)));
  CU(cudaMemcpy(h->d_tmask, mask.data(), 8 * mask.size(), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(h->d_tasrc, asrc.data(), 4 * asrc.size(), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(h->d_toff, T.off.data(), 4 * T.W, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(h->d_toffA, T.offA.data(), 4 * T.WA, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(h->d_tw2a, T.w2a.data(), T.W, cudaMemcpyHostToDevice));
  int gt = 1;  // (unused by the template trisolve; kept for introspection)
  h->G_tri = gt;
  return FASTILU_OK;
}

static TDev tdev(fastilu_handle h) {
  return TDev{h->T.W,   h->T.c0,    h->T.WA,  h->T.words, h->d_toff,
              h->d_toffA, h->d_tw2a, h->d_tmask, h->d_tasrc};
}

static fastilu_status create_impl(fastilu_handle h, int64_t n, const int64_t *row_ptr,
                                  const int32_t *col_idx, const double *values, int K) {
  const fastilu_options &o = h->opt;
  const bool multi = o.nranks > 1;
  h->n = n;
  h->K = K;
  h->row_begin = multi ? o.row_begin : 0;
  h->global_n = multi ? o.global_n : n;
  h->n_lead = multi ? o.n_lead : 0;
  if (multi) {
    if (o.global_n <= 0 || o.row_begin < 0 || o.row_begin + n > o.global_n || o.n_lead < 0 ||
        o.n_lead > o.row_begin || o.rank < 0 || o.rank >= o.nranks)
      FAIL(FASTILU_ERR_INVALID_ARG);
  }
  const int nt = hw_threads(o.num_threads);
  const int64_t g0 = h->row_begin - h->n_lead;
  const int64_t nrows = h->n_lead + n;
  const int64_t row_end = h->row_begin + n;
  int64_t bad = -1;
  int st = validate_csr(nrows, row_ptr, col_idx, g0, h->global_n, nt, &bad);
  if (st) {
    h->err_index = bad;
    return (fastilu_status)st;
  }
  const int64_t bw = half_bandwidth(nrows, row_ptr, col_idx, g0, nt);
  const int64_t o0 = multi ? std::max(g0, h->row_begin - (int64_t)(K + 1) * std::max<int64_t>(bw, 1))
                           : 0;
  Pattern pat;
  st = symbolic_iluk(nrows, row_ptr, col_idx, g0, o0, row_end, K, nt, pat, &bad);
  if (st) {
    h->err_index = bad;
    return (fastilu_status)st;
  }
  // ghost extents
  const int64_t own_r0 = h->row_begin - o0;  // pattern row index of the first owned row
  int64_t mincol = h->row_begin, maxcol = row_end - 1;
  for (int64_t r = own_r0; r < own_r0 + n; r++) {
    int64_t s = pat.rp[r], e = pat.rp[r + 1];
    if (e > s) {
      mincol = std::min<int64_t>(mincol, pat.ci[s]);
      maxcol = std::max<int64_t>(maxcol, pat.ci[e - 1]);
    }
  }
  h->G = h->row_begin - mincol;
  h->H = maxcol - (row_end - 1);
  if (!multi && (h->G != 0 || h->H != 0)) FAIL(FASTILU_ERR_BAD_MATRIX);
  // multi-GPU: whole 32-row slices of ghost rows (template-SELL layout), if the margin allows
  if (multi && h->G % 32 && (h->G + 31) / 32 * 32 <= own_r0) h->G = (h->G + 31) / 32 * 32;
  if (multi) {
    fastilu_status cs = comm_init(h->comm, h->opt, h->stream);
    if (cs) return cs;
  }
  if (h->G > own_r0) FAIL(FASTILU_ERR_UNSUPPORTED);  // ghost rows beyond the supplied margin
  h->lbase = h->row_begin - h->G;
  h->nloc = h->G + n;
  h->E = h->nloc + h->H;
  if (h->E >= (int64_t)INT32_MAX) FAIL(FASTILU_ERR_UNSUPPORTED);
  const int64_t lr0 = own_r0 - h->G;  // pattern row of local row 0
  const int64_t s_base = pat.rp[lr0];
  h->nnz_loc = pat.rp[own_r0 + n] - s_base;
  h->own_off = pat.rp[own_r0] - s_base;
  h->nnz_own = h->nnz_loc - h->own_off;
  // local structure
  std::vector<int64_t> rp(h->nloc + 1);
  std::vector<int32_t> ci(h->nnz_loc), dloc(h->nloc);
  int64_t m_max = 0, maxU = 0;
  for (int64_t r = 0; r <= h->nloc; r++) rp[r] = pat.rp[lr0 + r] - s_base;
  {
    std::vector<std::thread> th;
    int T = std::max(1, std::min<int>(nt, (int)(h->nloc / 4096 + 1)));
    std::vector<int64_t> mm(T, 0), mu(T, 0);
    for (int t = 0; t < T; t++)
      th.emplace_back([&, t]() {
        int64_t a = h->nloc * t / T, b = h->nloc * (t + 1) / T;
        for (int64_t r = a; r < b; r++) {
          const int64_t g = h->lbase + r;
          int32_t d = -1;
          for (int64_t p = rp[r]; p < rp[r + 1]; p++) {
            const int64_t c = pat.ci[s_base + p];
            ci[p] = (int32_t)(c - h->lbase);  // ghost rows may hold negative (unused) columns
            if (c == g) d = (int32_t)(p - rp[r]);
          }
          dloc[r] = d;
          mu[t] = std::max<int64_t>(mu[t], rp[r + 1] - rp[r] - d - 1);
          if (r >= h->G) mm[t] = std::max<int64_t>(mm[t], rp[r + 1] - rp[r]);
        }
      });
    for (auto &x : th) x.join();
    for (int t = 0; t < T; t++) {
      m_max = std::max(m_max, mm[t]);
      maxU = std::max(maxU, mu[t]);
    }
  }
  // host copies of the owned rows (introspection)
  h->h_rp.resize(n + 1);
  for (int64_t r = 0; r <= n; r++) h->h_rp[r] = pat.rp[own_r0 + r] - pat.rp[own_r0];
  h->h_ci.assign(pat.ci.begin() + pat.rp[own_r0], pat.ci.begin() + pat.rp[own_r0 + n]);
  h->h_lev.assign(pat.lev.begin() + pat.rp[own_r0], pat.lev.begin() + pat.rp[own_r0 + n]);
  // A layout for local rows [lbase, row_end): arp, adiag; owned rows: aci (local), apos
  const int64_t ar0 = h->lbase - g0;  // caller row index of local row 0
  h->a_in_off = row_ptr[ar0];
  h->a_in_nnz = row_ptr[nrows];
  h->nnzA_loc = row_ptr[ar0 + h->nloc] - h->a_in_off;
  std::vector<int64_t> arp(h->nloc + 1);
  std::vector<int32_t> adiag(h->nloc), aci(h->nnzA_loc, 0), apos(h->nnzA_loc, 0);
  for (int64_t r = 0; r <= h->nloc; r++) arp[r] = row_ptr[ar0 + r] - h->a_in_off;
  h->h_arp = arp;
  {
    std::vector<std::thread> th;
    int T = std::max(1, std::min<int>(nt, (int)(h->nloc / 4096 + 1)));
    std::vector<int> fail(T, 0);
    for (int t = 0; t < T; t++)
      th.emplace_back([&, t]() {
        int64_t a = h->nloc * t / T, b = h->nloc * (t + 1) / T;
        for (int64_t r = a; r < b; r++) {
          const int64_t g = h->lbase + r;
          const int64_t q0 = h->a_in_off + arp[r], q1 = h->a_in_off + arp[r + 1];
          for (int64_t q = q0; q < q1; q++)
            if (col_idx[q] == g) adiag[r] = (int32_t)(q - q0);
          int64_t p = rp[r];
          for (int64_t q = q0; q < q1; q++) {
            const int64_t c = col_idx[q] - h->lbase;
            while (p < rp[r + 1] && ci[p] < c) p++;
            if (p == rp[r + 1] || ci[p] != c) {
              fail[t] = 1;
              break;
            }
            aci[q - h->a_in_off] = (int32_t)c;
            apos[q - h->a_in_off] = (int32_t)(p - rp[r]);
          }
        }
      });
    for (auto &x : th) x.join();
    for (int t = 0; t < T; t++)
      if (fail[t]) FAIL(FASTILU_ERR_BAD_MATRIX);  // S must contain A (cannot happen)
  }
  int64_t nl_own = 0;
  for (int64_t r = h->G; r < h->nloc; r++) nl_own += dloc[r];
  const double nl_avg = n ? (double)nl_own / n : 1.0;
  const double u_avg = n ? (double)(h->nnz_own - n - nl_own) / n : 1.0;
  // block-dense patterns (3-dof elasticity type): block sweep with host-built term lists
  // (single GPU; measured faster than the template layout on these patterns)
  BlockPattern bp;
  if (!multi && !std::getenv("FASTILU_NO_BSR")) {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const int64_t max_terms = (int64_t)(fr / 4 / 8);  // term list <= a quarter of free memory
    h->bsr = build_blocks(rp, ci, h->nloc, nt, max_terms, bp);
  }
  // template-SELL fast path for structured patterns (else the CSR kernels below)
  {
    std::vector<unsigned long long> tmask;
    std::vector<int32_t> tasrc;
    bool ok = !h->bsr && !std::getenv("FASTILU_NO_TSELL") &&
              (!multi || (n % 32 == 0 && h->G % 32 == 0)) &&
              jit_available(nullptr) &&
              build_template(rp, ci, h->nloc, arp, aci, nt, h->T, tmask, tasrc);
    if (multi) {  // all ranks must agree on the layout (and on the template itself)
      std::vector<int64_t> all;
      fastilu_status cs = comm_allgather_i64(h->comm, {ok ? 1 : 0, ok ? (int64_t)h->T.hash : 0},
                                             all, h->stream);
      if (cs) return cs;
      for (int r = 0; r < h->opt.nranks; r++)
        if (!all[2 * r] || all[2 * r + 1] != all[1]) ok = false;
    }
    if (ok) {
      fastilu_status ts = setup_tsell(h, tmask, tasrc);
      if (ts == FASTILU_OK) h->tsell = true;
      else if (multi || ts != FASTILU_ERR_UNSUPPORTED) return ts;
    }
    if (h->tsell && K > 0) {  // nested level masks for the warm-up option
      std::vector<int8_t> llev(pat.lev.begin() + s_base, pat.lev.begin() + s_base + h->nnz_loc);
      for (int L = 0; L < K; L++) {
        std::vector<unsigned long long> lm;
        level_mask(rp, ci, llev, h->nloc, h->T, L, nt, lm);
        unsigned long long *d = nullptr;
        CU(dalloc(&d, (int64_t)lm.size()));
        CU(cudaMemcpy(d, lm.data(), 8 * lm.size(), cudaMemcpyHostToDevice));
        h->d_lmask.push_back(d);
      }
    }
  }
  // structure classes for the class-program sweep (falls back to the hash kernel if absent)
  ClassProgram cp;
  const bool have_prog = !h->tsell && !h->bsr &&
      !std::getenv("FASTILU_NO_CLASSES") &&
      build_classes(rp, ci, dloc, h->nloc, h->G, h->G + n, arp, apos, nt, (size_t)256 << 20,
                    1 << 16, cp);
  fastilu_status fs = h->tsell ? FASTILU_OK
                              : setup_configs(h, rp, ci, m_max, u_avg, nl_avg, maxU, have_prog, nt);
  if (fs && !(h->bsr && fs == FASTILU_ERR_UNSUPPORTED)) return fs;  // rows too long for smem
  if (h->bsr) {
    int gi = 4, gt = 1;
    while (gi < (double)h->nnz_own / std::max<int64_t>(h->n, 1) && gi < 32) gi *= 2;
    while (2 * gt < nl_avg && gt < 32) gt *= 2;
    h->G_init = gi;
    h->G_tri = gt;
    const int64_t st = (bp.bs * bp.bs + 1) & ~1;
    CU(dalloc(&h->d_bptr, bp.nb + 1));
    CU(dalloc(&h->d_brow, bp.nblk));
    CU(dalloc(&h->d_bcol, bp.nblk));
    CU(dalloc(&h->d_bdiag, bp.nb));
    CU(dalloc(&h->d_tptr, bp.nblk + 1));
    CU(cudaMalloc((void **)&h->d_terms, sizeof(int2) * (size_t)std::max<int64_t>(bp.nterms, 1)));
    for (int b = 0; b < 2; b++) {
      CU(dalloc(&h->d_vb[b], bp.nblk * st));
      CU(cudaMemset(h->d_vb[b], 0, sizeof(double) * bp.nblk * st));
    }
    CU(dalloc(&h->d_ahb, bp.nblk * st));
    CU(cudaMemset(h->d_ahb, 0, sizeof(double) * bp.nblk * st));  // fill entries: +0.0
    CU(cudaMemcpy(h->d_bptr, bp.bptr.data(), 8 * bp.bptr.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_brow, bp.brow.data(), 4 * bp.brow.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_bcol, bp.bcol.data(), 4 * bp.bcol.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_bdiag, bp.bdiag.data(), 4 * bp.bdiag.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_tptr, bp.tptr.data(), 8 * bp.tptr.size(), cudaMemcpyHostToDevice));
    if (bp.nterms)
      CU(cudaMemcpy(h->d_terms, bp.terms.data(), 4 * bp.terms.size(), cudaMemcpyHostToDevice));
    h->bsr_nterms = bp.nterms;
    h->B = BsrDev{bp.bs,     bp.nb,      bp.nblk,     h->d_bptr, h->d_brow,
                  h->d_bcol, h->d_bdiag, h->d_tptr,   h->d_terms};
    // options measured on the Table-6 problem and 3-dof 48^3 ILU(1/2): staging
    // the tile's block rows in shared memory (FASTILU_BSR_SMEM_KB) costs L1 capacity and is
    // slower, so off; 4 resident CTAs (64 registers, FASTILU_BSR_MINB) beat 3 (80 registers).
    const char *sk = std::getenv("FASTILU_BSR_SMEM_KB");
    h->bsr_smem = (size_t)(sk ? atoi(sk) : 0) * 1024;
    const char *mb = std::getenv("FASTILU_BSR_MINB");
    h->bsr_minb = mb ? atoi(mb) : 4;
    int bps = 0;
    if (bsr_sweep_occupancy(bp.bs, h->bsr_threads, h->bsr_smem, h->bsr_minb, &bps) !=
            cudaSuccess || bps < 1)
      return FASTILU_ERR_CUDA;
    h->bsr_grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((int64_t)sm_count(h->device) * bps,
                             (bp.nblk + h->bsr_threads - 1) / h->bsr_threads));
    h->scfg.grid = std::max(h->scfg.grid, h->bsr_grid);  // partials capacity
  }
  if (h->scfg.prog) {
    h->nclasses = cp.nclasses;
    CU(dalloc(&h->d_rclass, (int64_t)cp.row_class.size()));
    CU(dalloc(&h->d_coff, (int64_t)cp.class_off.size()));
    CU(dalloc(&h->d_caoff, (int64_t)cp.class_aoff.size()));
    CU(dalloc(&h->d_prog, (int64_t)cp.prog.size()));
    CU(cudaMemcpy(h->d_rclass, cp.row_class.data(), 4 * cp.row_class.size(),
                  cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_coff, cp.class_off.data(), 8 * cp.class_off.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_caoff, cp.class_aoff.data(), 4 * cp.class_aoff.size(),
                  cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_prog, cp.prog.data(), cp.prog.size(), cudaMemcpyHostToDevice));
  }
  // device allocations
  if (!h->tsell) {  // CSR structure of S (the template path needs none)
    CU(dalloc(&h->d_rp, h->nloc + 1));
    CU(dalloc(&h->d_ci, h->nnz_loc));
    CU(dalloc(&h->d_dloc, h->nloc));
    CU(dalloc(&h->d_apos, h->nnzA_loc));
    CU(dalloc(&h->d_ahat, h->nnzA_loc));  // ahat on A's pattern (ghost rows' stay 0)
    CU(cudaMemset(h->d_ahat, 0, sizeof(double) * h->nnzA_loc));
    CU(dalloc(&h->d_partials, std::max<int64_t>(h->scfg.grid, kSumsqBlocks)));
    for (int b = 0; b < 2; b++) CU(dalloc(&h->d_vals[b], h->nnz_loc));
  }
  CU(dalloc(&h->d_arp, h->nloc + 1));
  CU(dalloc(&h->d_aci, h->nnzA_loc));  // A's local columns (CSR init, GMRES SpMV)
  CU(dalloc(&h->d_adiag, h->nloc));
  CU(dalloc(&h->d_aval, h->nnzA_loc));
  for (int b = 0; b < 2; b++) {
    CU(dalloc(&h->d_ud[b], h->E));
    CU(dalloc(&h->d_z[b], h->E));
    CU(dalloc(&h->d_w[b], h->E));
  }
  CU(dalloc(&h->d_s, h->E));
  CU(dalloc(&h->d_ad, h->E));
  CU(dalloc(&h->d_y, h->E));
  CU(dalloc(&h->d_err, 1));
  CU(cudaMallocHost((void **)&h->h_err, sizeof(ErrFlags)));
  if (!h->tsell) {
    CU(cudaMemcpy(h->d_rp, rp.data(), sizeof(int64_t) * rp.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_ci, ci.data(), sizeof(int32_t) * ci.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_dloc, dloc.data(), sizeof(int32_t) * dloc.size(),
                  cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_apos, apos.data(), sizeof(int32_t) * apos.size(),
                  cudaMemcpyHostToDevice));
  }
  CU(cudaMemcpy(h->d_aci, aci.data(), sizeof(int32_t) * aci.size(), cudaMemcpyHostToDevice));
  {
    const double a_avg = n ? (double)(arp[h->nloc] - arp[h->G]) / (double)n : 1.0;
    int gs = 4;
    while (gs < a_avg && gs < 32) gs *= 2;
    h->G_spmv = gs;
  }
  CU(cudaMemcpy(h->d_arp, arp.data(), sizeof(int64_t) * arp.size(), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(h->d_adiag, adiag.data(), sizeof(int32_t) * adiag.size(),
                cudaMemcpyHostToDevice));
  CU(cudaMemset(h->d_s, 0, sizeof(double) * h->E));
  CU(cudaMemset(h->d_ad, 0, sizeof(double) * h->E));
  for (int b = 0; b < 2; b++) {
    CU(cudaMemset(h->d_ud[b], 0, sizeof(double) * h->E));
    CU(cudaMemset(h->d_z[b], 0, sizeof(double) * h->E));
    CU(cudaMemset(h->d_w[b], 0, sizeof(double) * h->E));
  }
  for (int i = 0; i < 6; i++) CU(cudaEventCreate(&h->ev[i]));
  if (multi) {
    int64_t nl_global = 0;
    fastilu_status cs = comm_layout(h->comm, h->row_begin, h->n, h->G, h->H, rp.data(), nl_own,
                                    &nl_global, h->tsell ? h->T.W : 0,
                                    h->tsell ? h->T.hash : 0, h->stream);
    if (cs) return cs;
    const double nlg = (double)nl_global / (double)std::max<int64_t>(h->global_n, 1);
    int gt = 1;  // same rule as setup_configs, from the GLOBAL average (partition-independent)
    while (2 * gt < nlg && gt < 32) gt *= 2;
    h->G_tri = gt;
  }
  if (values) return upload_values(h, values, false);
  return FASTILU_OK;
}

extern "C" fastilu_status fastilu_create(fastilu_handle *out, int64_t n, const int64_t *row_ptr,
                                         const int32_t *col_idx, const double *values,
                                         int level_k, const fastilu_options *opts) {
  if (!out) FAIL(FASTILU_ERR_INVALID_ARG);
  *out = nullptr;
  DeviceGuard dg_(-1);  // restores the caller's device (create switches to opts->device)
  fastilu_handle h = new (std::nothrow) fastilu_handle_s();
  if (!h) return FASTILU_ERR_OOM;
  *out = h;
  if (opts) h->opt = *opts; else fastilu_default_options(&h->opt);
  if (n < 0 || !row_ptr || (n > 0 && !col_idx) || level_k < 0 || level_k > 127 ||
      h->opt.nranks < 1 || !(h->opt.omega > 0.0 && h->opt.omega <= 1.0) ||
      !(h->opt.omega_tri > 0.0 && h->opt.omega_tri <= 1.0) || !(h->opt.shift >= 0.0))
    FAIL(FASTILU_ERR_INVALID_ARG);
  if (h->opt.device >= 0) {
    if (cudaSetDevice(h->opt.device) != cudaSuccess) return FASTILU_ERR_CUDA;
    h->device = h->opt.device;
  } else {
    if (cudaGetDevice(&h->device) != cudaSuccess) return FASTILU_ERR_CUDA;
  }
  if (h->opt.stream) {
    h->stream = (cudaStream_t)h->opt.stream;
  } else {
    if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess)
      return FASTILU_ERR_CUDA;
    h->own_stream = true;
  }
  return create_impl(h, n, row_ptr, col_idx, values, level_k);
}

extern "C" fastilu_status fastilu_set_values(fastilu_handle h, const double *values) {
  if (!h || !values || !h->d_aval) FAIL(FASTILU_ERR_INVALID_ARG);
  DeviceGuard dg_(h->device);
  return upload_values(h, values, false);
}

extern "C" fastilu_status fastilu_set_values_device(fastilu_handle h, const double *values) {
  if (!h || !values || !h->d_aval) FAIL(FASTILU_ERR_INVALID_ARG);
  DeviceGuard dg_(h->device);
  return upload_values(h, values, true);
}

// --------------------------------------------------------------------------- compute
// nsweeps synchronous sweeps; with rtol > 0, stop after the first sweep s whose residual of
// iterate s-1 satisfies r(s-1) <= rtol ||Ahat|_S||_F (reading G15), at most nsweeps.
static fastilu_status compute_impl(fastilu_handle h, int nsweeps, double rtol, int *done,
                                   bool warmup = false, bool async = false) {
  if (!h || nsweeps < 0) FAIL(FASTILU_ERR_INVALID_ARG);
  if (async) {  // in-place variants (single GPU): template kernel or block kernel
    if (!(h->tsell || h->bsr) || h->comm) FAIL(FASTILU_ERR_UNSUPPORTED);
    if (h->tsell) {
      // "Block Size": each thread updates a contiguous block of ~ept targets of
      // its row; parts = W / ept rounded up to a divisor of the block's warps
      const int warps = h->t_threads / 32;
      const int ept = h->async_ept > 0 ? h->async_ept : (h->T.W + h->t_parts - 1) / h->t_parts;
      int parts = 1;
      while (parts < warps && (h->T.W + parts - 1) / parts > ept) parts *= 2;
      void *fn = nullptr;
      for (auto &pr : h->jit_async)
        if (pr.first == parts) fn = pr.second;
      if (!fn) {
        std::string log;
        const std::string src = sweep_source(h->T, h->t_threads, parts, 0, true, false, false,
                                             true);
        if (jit_get(src, "fastilu_tsell_sweep_async", h->device, &fn, &log))
          FAIL(FASTILU_ERR_UNSUPPORTED);
        h->jit_async.push_back({parts, fn});
      }
      h->jit_sweep_async = fn;
      h->async_parts = parts;
      h->async_rows = 32 * (warps / parts);
    }
  }
  const int per_level = nsweeps;
  if (warmup) {  // FastILU(0), ..., FastILU(K) with nsweeps each
    if (!h->tsell && h->K > 0) FAIL(FASTILU_ERR_UNSUPPORTED);
    nsweeps = per_level * (h->K + 1);
  }
  if (!h->have_values || !h->d_aval) FAIL(FASTILU_ERR_STATE);
  DeviceGuard dg_(h->device);
  (void)cudaGetLastError();  // clear a non-sticky error left by the caller's own CUDA work
  h->computed = false;
  h->err_index = -1;
  cudaStream_t st = h->stream;
  if (nsweeps > h->hist_cap) {
    if (h->d_r2) cudaFree(h->d_r2);
    if (h->h_r2) cudaFreeHost(h->h_r2);
    h->d_r2 = nullptr;
    h->h_r2 = nullptr;
    CU(dalloc(&h->d_r2, nsweeps));
    CU(cudaMallocHost((void **)&h->h_r2, sizeof(double) * nsweeps));
    h->hist_cap = nsweeps;
  }
  CU(cudaMemsetAsync(h->d_err, 0xff, sizeof(ErrFlags), st));
  DevPattern P{h->d_rp, h->d_ci, h->d_dloc};
  const int64_t r0 = h->G, r1 = h->G + h->n;
  CU(cudaEventRecord(h->ev[0], st));
  // a2: scaling for every local row (lower ghosts included), then the upper ghosts' s / ad
  if (h->tsell && h->jit_scale) {  // from the diagonal column of A's template copy
    const double *aT = h->d_aT;
    long long z0 = 0, nl = h->nloc;
    double *sp = h->d_s, *adp = h->d_ad, sh = h->opt.shift;
    ErrFlags *ep = h->d_err;
    void *args[] = {&aT, &z0, &nl, &sp, &adp, &ep, &sh};
    if (jit_launch(h->jit_scale, (int)((h->nloc + 255) / 256), 256, st, args))
      FAIL(FASTILU_ERR_CUDA);
  } else {
    CU(launch_scale(h->d_arp, h->d_adiag, h->d_aval, 0, h->nloc, h->d_s, h->d_ad, h->d_err,
                    h->opt.shift, st));
  }
  if (h->comm) {  // lower ghosts' s / ahat_ii are computed locally from the lead rows of A
    fastilu_status cs = comm_vector_halo(h->comm, h->d_s, st, false, true);
    if (cs) return cs;
  }
  // a3: ahat and the initial guess (iterate 0) for the owned rows.  With the fused first
  // sweep, iterate 0 is computed from ahat inside sweep 1 and never stored.
  // Multi-GPU: the lower ghost rows' diagonal and upper ahat are computed locally (their A
  // rows and scales are local), so sweep 1 stages them like owned rows and iterate 0 needs no
  // halo.
  const bool fuse_init = h->tsell && h->jit_st_init && h->jit_st && h->jit_ahat && !warmup &&
                         !async && nsweeps >= 1 && h->opt.omega == 1.0;
  if (h->tsell && fuse_init) {
    const double *aT = h->d_aT, *sv = h->d_s;
    const unsigned long long *mk = h->d_tmask;
    long long a0 = 0, a1 = r1, aown = r0;
    double *hp = h->d_ahat, sh = h->opt.shift;
    ErrFlags *ep = h->d_err;
    void *args[] = {&aT, &sv, &mk, &a0, &a1, &hp, &ep, &sh, &aown};
    if (r1 > 0 && jit_launch(h->jit_ahat, (int)((r1 + 255) / 256), 256, st, args))
      FAIL(FASTILU_ERR_CUDA);
  } else if (h->tsell) {
    CU(launch_tsell_init(tdev(h), h->d_aT, h->d_s, h->d_ad, r0, r1, h->d_ahat, h->d_vals[0],
                         h->d_ud[0], h->d_err, h->opt.shift, st, !fuse_init));
  }
  else
    CU(launch_init(P, h->d_arp, h->d_aci, h->d_apos, h->d_aval, h->d_s, h->d_ad, r0, r1,
                   h->d_ahat, h->d_vals[0], h->d_ud[0], h->d_err, h->G_init, h->opt.shift, st));
  if (h->bsr) {  // iterate 0 and ahat into the block layout
    CU(launch_bsr_from_csr(h->B, h->d_rp, h->d_vals[0], h->d_vb[0], h->n, st));
    CU(launch_bsr_ahat(h->B, h->d_arp, h->d_apos, h->d_ahat, h->d_ahb, h->n, st));
  }
  CU(cudaEventRecord(h->ev[1], st));
  double thr2 = -1.0;  // (rtol ||Ahat|_S||_F)^2, tolerance mode only
  std::vector<double> r2tol;
  if (rtol > 0.0) {
    // owned rows only (with the fused first sweep the lower ghosts' ahat is stored too; G is
    // a whole number of slices on the template path)
    const int64_t a_off = h->tsell ? (h->G / 32) * h->T.WA * 32 : 0;
    const int64_t na = h->tsell ? h->nsl * h->T.WA * 32 - a_off : h->nnzA_loc;
    CU(launch_sumsq(h->d_ahat + a_off, na, h->d_partials, h->d_r2, st));
    double a2 = 0.0;
    CU(cudaMemcpyAsync(h->h_r2, h->d_r2, sizeof(double), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    a2 = h->h_r2[0];
    if (h->comm) {
      ErrFlags dummy{~0ull, ~0ull};
      fastilu_status cs = comm_allreduce_host(h->comm, &a2, 1, dummy);
      if (cs) return cs;
    }
    thr2 = rtol * rtol * a2;
  }
  int executed = 0;
  // a4/a5: nsweeps synchronous sweeps, ping-pong buffers
  for (int sw = 1; sw <= nsweeps; sw++) {
    if (sw == 2) CU(cudaEventRecord(h->ev[5], st));  // sweep 1 / the rest split
    executed = sw;
    const int ib_async = 0;  // asynchronous sweeps stay in buffer 0 (in place)
    if (thr2 >= 0.0 && sw > 1) {  // r(sw-2) of the previous sweep decides whether to go on
      CU(cudaMemcpyAsync(h->h_r2 + (sw - 2), h->d_r2 + (sw - 2), sizeof(double),
                         cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
      double v = h->h_r2[sw - 2];
      if (h->comm) {
        ErrFlags dummy{~0ull, ~0ull};
        fastilu_status cs = comm_allreduce_host(h->comm, &v, 1, dummy);
        if (cs) return cs;
      }
      r2tol.push_back(v);
      if (v <= thr2) {
        executed = sw - 1;
        break;
      }
    }
    const int ib = async ? ib_async : (sw - 1) & 1, ob = async ? ib_async : sw & 1;
    // multi-GPU template path: the factor halo (diagonal + strict-upper columns of the ghost
    // rows, packed) flies on the comm stream while the rows that read no ghost row are swept;
    // the first `bnd` owned rows (pivot rows reach below them into the ghosts) follow
    cudaEvent_t halo_done = nullptr;
    int64_t bnd = 0;
    if (h->comm && !(sw == 1 && fuse_init)) {  // fused sweep 1 reads no stored iterate 0
      fastilu_status cs =
          h->tsell ? comm_factor_halo_upper(h->comm, h->d_vals[ib], h->d_ud[ib], h->T.W,
                                            h->T.c0, st, &halo_done)
                   : comm_factor_halo(h->comm, h->d_vals[ib], h->d_rp, h->d_ud[ib], st);
      if (cs) return cs;
      if (halo_done) {
        bnd = std::min<int64_t>(h->n, (-(int64_t)h->T.off[0] + 31) / 32 * 32);
        if (std::getenv("FASTILU_NO_HALO_OVERLAP")) bnd = h->n;
      }
    }
    SweepArgs sa{P,           h->d_arp,      h->d_apos,     h->d_ahat, h->d_vals[ib],
                 h->d_vals[ob], h->d_ud[ib], h->d_ud[ob], r0,        r1,
                 h->opt.omega,  h->d_partials, h->d_err};
    if (h->tsell) {
      const double *old = h->d_vals[ib], *ahat = h->d_ahat, *udo = h->d_ud[ib];
      double *outp = h->d_vals[ob], *udn = h->d_ud[ob];
      const unsigned long long *mk = h->d_tmask;
      if (warmup && per_level > 0) {
        const int lvl = (sw - 1) / per_level;
        if (lvl < h->K) mk = h->d_lmask[lvl];
      }
      double om = h->opt.omega;
      unsigned long long *zp = &h->d_err->zero_pivot;
      int sstr = h->t_sstride;
      const bool staged = h->jit_st && !async;
      void *fn = nullptr;
      int smem = 0, grid = 0, thr = 0;
      int64_t rows_tile = 0;
      void *tm0 = nullptr, *tm1 = nullptr;
      if (staged) {
        fn = (sw == 1 && !warmup && h->jit_st_first) ? h->jit_st_first : h->jit_st;
        smem = h->st.smem, grid = h->st_grid, thr = h->st.threads, rows_tile = h->st.rows;
        tm0 = h->st_tmap[ib].b, tm1 = h->st_tmap_own[ib].b;
        if (sw == 1 && fuse_init) {
          fn = h->jit_st_init;
          smem = h->st_init.smem, grid = h->st_init_grid, thr = h->st_init.threads;
          rows_tile = h->st_init.rows;
          tm0 = h->st_tmap_ahat.b, tm1 = h->st_tmap_own_ahat.b;
        }
      } else {
        fn = async ? h->jit_sweep_async
             : (sw == 1 && !warmup && h->jit_sweep_first) ? h->jit_sweep_first
                                                          : h->jit_sweep;
        grid = h->t_grid, thr = h->t_threads;
      }
      // one launch over local rows [a0, a1) with its own tile counter and partials; returns the
      // number of tiles (partials written) or -1
      auto sweep_range = [&](int64_t b0, int64_t b1, unsigned int *ctr, double *part) -> int64_t {
        if (b1 <= b0) return 0;
        long long a0 = b0, a1 = b1;
        int64_t ntl;
        if (staged) {
          ntl = (b1 - b0 + rows_tile - 1) / rows_tile;
          void *sargs[] = {&old, &outp, &ahat, &mk, &udn, &a0, &a1, &om, &part, &zp, &ctr,
                           tm0, tm1};
          if (jit_launch_smem(fn, (int)std::min<int64_t>(grid, ntl), thr, smem, st, sargs))
            return -1;
        } else if (async) {
          ntl = (b1 - b0 + h->async_rows - 1) / h->async_rows;
          int one = 1;
          void *args[] = {&old, &outp, &ahat, &mk, &udo, &udn, &a0, &a1, &om, &part, &zp, &ctr,
                          &one};
          if (jit_launch(fn, (int)std::min<int64_t>(grid, ntl), thr, st, args)) return -1;
        } else {
          const int64_t spt = h->t_rows_tile / 32, ss = h->t_sstride;
          ntl = ((b1 - b0 + 31) / 32 + spt * ss - 1) / (spt * ss) * ss;
          void *args[] = {&old, &outp, &ahat, &mk, &udo, &udn, &a0, &a1, &om, &part, &zp, &ctr,
                          &sstr};
          if (jit_launch(fn, (int)std::min<int64_t>(grid, ntl), thr, st, args)) return -1;
        }
        return ntl;
      };
      if (!halo_done) {
        const int64_t nt = sweep_range(r0, r1, h->d_counter, h->d_partials);
        if (nt < 0) return FASTILU_ERR_CUDA;
        CU(launch_reduce_reset(h->d_partials, (int)nt, h->d_r2 + (sw - 1), h->d_counter, st));
        continue;
      }
      const int64_t nt1 = sweep_range(r0 + bnd, r1, h->d_counter, h->d_partials);
      if (nt1 < 0) return FASTILU_ERR_CUDA;
      CU(cudaStreamWaitEvent(st, halo_done, 0));
      const int64_t nt2 = sweep_range(r0, r0 + bnd, h->d_counter + 1, h->d_partials + nt1);
      if (nt2 < 0) return FASTILU_ERR_CUDA;
      CU(launch_reduce_reset(h->d_partials, (int)(nt1 + nt2), h->d_r2 + (sw - 1), h->d_counter,
                             st));
      CU(cudaMemsetAsync(h->d_counter + 1, 0, sizeof(unsigned int), st));
      continue;
    }
    if (h->bsr && async) {  // nb consecutive target blocks per thread, in place
      const int bb = h->B.bs * h->B.bs;
      const int nb = std::max(1, (h->async_ept > 0 ? h->async_ept : bb) / bb);
      const int64_t nthr = (h->B.nblk + nb - 1) / nb;
      const int grid = (int)std::max<int64_t>(  // <= bsr_grid: the partials' capacity
          1, std::min<int64_t>((nthr + 255) / 256, (int64_t)h->bsr_grid));
      CU(launch_bsr_sweep_async(h->B, h->d_ahb, h->d_vb[0], h->opt.omega, h->d_partials,
                                h->d_err, grid, nb, st));
      CU(launch_reduce(h->d_partials, grid, h->d_r2 + (sw - 1), st));
      continue;
    }
    if (h->bsr) {
      CU(launch_bsr_sweep(h->B, h->d_ahb, h->d_vb[ib], h->d_vb[ob], h->opt.omega, h->d_partials,
                          h->d_err, h->bsr_grid, h->bsr_threads, h->bsr_smem, h->bsr_minb,
                          st));
      CU(launch_reduce(h->d_partials, h->bsr_grid, h->d_r2 + (sw - 1), st));
      continue;
    }
    if (h->scfg.prog) {
      ProgView pv{h->d_rclass, h->d_coff, h->d_caoff, h->d_prog};
      CU(launch_sweep_prog(sa, pv, h->scfg, st));
    } else {
      CU(launch_sweep(sa, h->scfg, st));
    }
    CU(launch_reduce(h->d_partials, h->scfg.grid, h->d_r2 + (sw - 1), st));
  }
  nsweeps = executed;
  if (done) *done = executed;
  if (h->bsr) {  // factors back to S row order (+ u_ii) for apply / get_factors
    const int fb = async ? 0 : (nsweeps & 1);
    CU(launch_bsr_to_csr(h->B, h->d_rp, h->d_vb[fb], h->d_vals[fb], h->d_ud[fb], h->n, st));
  }
  CU(cudaEventRecord(h->ev[2], st));
  CU(cudaMemcpyAsync(h->h_err, h->d_err, sizeof(ErrFlags), cudaMemcpyDeviceToHost, st));
  if (nsweeps)
    CU(cudaMemcpyAsync(h->h_r2, h->d_r2, sizeof(double) * nsweeps, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  CU(cudaEventElapsedTime(&h->t_init, h->ev[0], h->ev[1]));
  CU(cudaEventElapsedTime(&h->t_sweeps, h->ev[1], h->ev[2]));
  h->t_sweep1 = h->t_sweeps;
  h->last_ns = executed;
  if (executed >= 2) CU(cudaEventElapsedTime(&h->t_sweep1, h->ev[1], h->ev[5]));
  h->resid.assign(nsweeps, 0.0);
  std::vector<double> r2(h->h_r2, h->h_r2 + nsweeps);
  ErrFlags ef = *h->h_err;  // local rows -> global rows
  if (ef.zero_diag != ~0ull) ef.zero_diag += (unsigned long long)h->lbase;
  if (ef.zero_pivot != ~0ull) ef.zero_pivot += (unsigned long long)h->lbase;
  if (h->comm) {
    fastilu_status cs = comm_allreduce_host(h->comm, r2.data(), (int)r2.size(), ef);
    if (cs) return cs;
  }
  for (size_t q = 0; q < r2tol.size() && q < r2.size(); q++) r2[q] = r2tol[q];
  for (int i = 0; i < nsweeps; i++) h->resid[i] = std::sqrt(r2[i]);
  h->cur = async ? 0 : (nsweeps & 1);
  h->vals_cur = h->d_vals[h->cur];
  h->ud_cur = h->d_ud[h->cur];
  if (ef.zero_diag != ~0ull) {
    h->err_index = (int64_t)ef.zero_diag;
    return FASTILU_ERR_ZERO_DIAG;
  }
  if (ef.zero_pivot != ~0ull) {
    h->err_index = (int64_t)ef.zero_pivot;
    return FASTILU_ERR_ZERO_PIVOT;
  }
  h->computed = true;
  return FASTILU_OK;
}

static fastilu_status apply_impl(fastilu_handle h, const double *b, double *x, int ntri);
static int jit_jacobi(fastilu_handle h, bool lower, const double *vals, const double *ud,
                      const double *rhs, const double *xo, double *xn, double *xf, int64_t r0,
                      int64_t r1, int64_t Gh, double om, bool final_x);

// fastilu_compute_host: new values from host memory + nsweeps sweeps, the upload pipelined with
// the compute.  Chunks of >= A's bandwidth rows: chunk c's values go up on a copy stream; on
// the compute stream chunk c is gathered and scaled, chunk c-1 gets ahat (its s neighbours now
// exist), and the sweeps advance along a diagonal (step d: sweep s on chunk d-s+1, s ascending),
// which keeps every iterate a later chunk still reads alive in the two ping-pong buffers: sweep
// s of chunk c reads iterate s-1 of rows <= its own only.  Same kernels, same per-entry
// arithmetic as set_values + compute; only the residual's sum is taken per chunk.
//
// With nsweeps <= 3 every factor iterate has its own buffer and all sweeps of a chunk run at
// once (no diagonal).  With x_host (solve_host; FASTILU_SOLVE_NOPIPE=1 runs the apply after the
// compute instead), the apply rides the same pipeline: b goes up chunk by chunk behind the
// values, a chunk's L Jacobi sweeps run as soon as its factors are final and the U sweeps follow
// their dependency cone right behind (one buffer per Jacobi iterate), each chunk's x copied back
// as soon as its last U sweep is done.  Same kernels, rows and order of terms as apply: x is
// bitwise the same.
static fastilu_status compute_host_impl(fastilu_handle h, const double *values, int nsweeps,
                                        const double *b_host = nullptr,
                                        bool *b_queued = nullptr, double *x_host = nullptr,
                                        int ntri = 0, bool *x_done = nullptr) {
  if (b_queued) *b_queued = false;
  if (x_done) *x_done = false;
  const int64_t R = h->st.rows > 0 ? h->st.rows : 256;
  int64_t bwA = 0;
  for (int32_t o : h->T.offA) bwA = std::max<int64_t>(bwA, std::abs((int64_t)o));
  for (int32_t o : h->T.off) bwA = std::max<int64_t>(bwA, std::abs((int64_t)o));  // S's band
  int64_t chunk = std::max<int64_t>(bwA, 16 * R);
  chunk = std::max<int64_t>(chunk, (h->n + 15) / 16);
  chunk = (chunk + R - 1) / R * R;
  // chunk boundaries: equal chunks, the last one cut into up to 4 pieces of at least the band
  // (FASTILU_SOLVE_TAIL overrides the 4), so that less work waits for the last bytes (c4 e2e:
  // 76.2 -> 74.3 ms, profiles/r2ze_e2e_pipeline_ab.log)
  std::vector<int64_t> bnd;
  for (int64_t r = 0; r < h->n; r += chunk) bnd.push_back(r);
  {
    const char *te = std::getenv("FASTILU_SOLVE_TAIL");
    const int64_t last = bnd.back(), rows = h->n - last;
    const int64_t minp = (std::max<int64_t>(bwA, R) + R - 1) / R * R;
    const int64_t pieces =
        std::max<int64_t>(1, std::min<int64_t>(te ? std::atoi(te) : 4, rows / minp));
    const int64_t step = (rows / pieces + R - 1) / R * R;
    for (int64_t q = 1; q < pieces && last + q * step < h->n; q++) bnd.push_back(last + q * step);
  }
  bnd.push_back(h->n);
  const int C = (int)bnd.size() - 1;
  // staged template sweeps (init fused into sweep 1), or the register-pivot template sweeps
  // (narrow templates: iterate 0 stored by the init kernel, diagonal schedule)
  const bool staged_ok = h->jit_st && h->jit_st_init && h->jit_ahat && h->st.shift == 0;
  const bool regp = !staged_ok && h->jit_sweep != nullptr;
  const bool ok = h->tsell && !h->comm && (staged_ok || regp) && h->jit_scale && nsweeps >= 1 &&
                  h->opt.omega == 1.0 && h->G == 0 && C >= 2 &&
                  !std::getenv("FASTILU_NO_PIPELINE");
  if (!ok) {
    fastilu_status us = upload_values(h, values, false);
    if (us) return us;
    return compute_impl(h, nsweeps, 0.0, nullptr);
  }
  h->computed = false;
  h->have_values = false;  // d_aval is overwritten below; set again once every chunk landed
  h->err_index = -1;
  cudaStream_t st = h->stream;
  if (!h->copy_stream) CU(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
  while ((int)h->chunk_ev.size() < C + 1) {
    cudaEvent_t e;
    // FASTILU_TRACE=1 (diagnostic): timed chunk events, printed by solve_host
    CU(cudaEventCreateWithFlags(&e, std::getenv("FASTILU_TRACE") ? cudaEventDefault
                                                                 : cudaEventDisableTiming));
    h->chunk_ev.push_back(e);
  }
  if (nsweeps > h->hist_cap) {
    if (h->d_r2) cudaFree(h->d_r2);
    if (h->h_r2) cudaFreeHost(h->h_r2);
    h->d_r2 = nullptr;
    h->h_r2 = nullptr;
    CU(dalloc(&h->d_r2, nsweeps));
    CU(cudaMallocHost((void **)&h->h_r2, sizeof(double) * nsweeps));
    h->hist_cap = nsweeps;
  }
  if (C * nsweeps > h->r2c_cap) {
    if (h->d_r2c) cudaFree(h->d_r2c);
    h->d_r2c = nullptr;
    CU(dalloc(&h->d_r2c, (int64_t)C * nsweeps));
    h->r2c_cap = C * nsweeps;
  }
  auto rb = [&](int c) { return bnd[c]; };
  // FASTILU_DEBUG_SYNC=1: synchronise after every step of the pipeline and name a failing one
  static const bool dbg_sync = std::getenv("FASTILU_DEBUG_SYNC") != nullptr;
  auto dbg = [&](const char *what, int a, int b2) -> fastilu_status {
    if (!dbg_sync) return FASTILU_OK;
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      fprintf(stderr, "fastilu: %s after %s (%d, %d)\n", cudaGetErrorString(e), what, a, b2);
      return FASTILU_ERR_CUDA;
    }
    return FASTILU_OK;
  };

  CU(cudaMemsetAsync(h->d_err, 0xff, sizeof(ErrFlags), st));
  CU(cudaEventRecord(h->ev[0], st));
  // every chunk's values up front on the copy stream, ordered after the compute stream's
  // previous work (the previous compute may still read d_aval / d_aT)
  CU(cudaEventRecord(h->ev[1], st));
  CU(cudaStreamWaitEvent(h->copy_stream, h->ev[1], 0));
  // The buffers this call adds are allocated before its uploads and kernels are queued; without
  // the memory for them it falls back (to the diagonal / to the apply after the compute).
  // nodiag (nsweeps <= 3): every iterate of the sweeps has its own buffer -- iterate s in
  // buffer bufi[s] (the last in d_vals[nsweeps & 1] as after compute; a third iterate buffer
  // for nsweeps = 3) -- so all sweeps of chunk k run as soon as its Â is known, instead of along
  // the diagonal the two ping-pong buffers need (FASTILU_SOLVE_DIAG=1: the diagonal)
  bool nodiag = nsweeps <= 3 && !regp && !std::getenv("FASTILU_SOLVE_DIAG");
  if (nodiag && nsweeps == 3 && !h->d_vals3) {
    const int64_t nv = h->nsl * h->T.W * 32;
    if (dalloc(&h->d_vals3, nv) != cudaSuccess ||
        dalloc(&h->d_ud3, std::max<int64_t>(h->nsl * 32, 1)) != cudaSuccess) {
      (void)cudaGetLastError();
      if (h->d_vals3) cudaFree(h->d_vals3);
      h->d_vals3 = nullptr;
      h->d_ud3 = nullptr;
      nodiag = false;
    } else {
      CU(cudaMemsetAsync(h->d_vals3, 0, sizeof(double) * nv, st));  // absent slots stay +0.0
      const bool cm = h->st.colmajor != 0;
      if ((cm ? jit_tmap_sell_cm : jit_tmap_sell)(h->st_tmap3.b, h->d_vals3, h->T.W, h->nsl,
                                                  h->st.box_cols, h->st.box_slices) ||
          (cm ? jit_tmap_sell_cm : jit_tmap_sell)(h->st_tmap_own3.b, h->d_vals3, h->T.W,
                                                  h->nsl, std::max(1, h->st.own_cols),
                                                  h->st.rows / 32))
        FAIL(FASTILU_ERR_CUDA);
    }
  }
  bool pipe_x = b_host && x_host && ntri >= 1 && h->jit_jac[0] && h->jit_jac[1];
  if (pipe_x && h->it_cap < ntri) {  // one buffer per Jacobi iterate
    if (h->d_it) cudaFree(h->d_it);
    h->d_it = nullptr;
    h->it_cap = 0;
    if (dalloc(&h->d_it, (int64_t)2 * ntri * std::max<int64_t>(h->n, 1)) != cudaSuccess) {
      (void)cudaGetLastError();
      h->d_it = nullptr;
      pipe_x = false;
    } else {
      h->it_cap = ntri;
    }
  }
  if (pipe_x) {
    if (!h->d_bx) CU(dalloc(&h->d_bx, 2 * h->n));
    while ((int)h->x_ev.size() < C) {
      cudaEvent_t e;
      CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      h->x_ev.push_back(e);
    }
  }
  for (int c = 0; c < C; c++) {
    const int64_t a0 = h->h_arp[rb(c)], a1 = h->h_arp[rb(c + 1)];
    if (a1 > a0)
      CU(cudaMemcpyAsync(h->d_aval + a0, values + h->a_in_off + a0, sizeof(double) * (a1 - a0),
                         cudaMemcpyHostToDevice, h->copy_stream));
    if (pipe_x)  // chunk c of b behind chunk c of the values
      CU(cudaMemcpyAsync(h->d_bx + rb(c), b_host + rb(c), sizeof(double) * (rb(c + 1) - rb(c)),
                         cudaMemcpyHostToDevice, h->copy_stream));
    CU(cudaEventRecord(h->chunk_ev[c], h->copy_stream));
  }
  if (b_host && !pipe_x) {  // solve_host: the right-hand side follows the values
    if (!h->d_bx) CU(dalloc(&h->d_bx, 2 * h->n));
    CU(cudaMemcpyAsync(h->d_bx, b_host, sizeof(double) * h->n, cudaMemcpyHostToDevice,
                       h->copy_stream));
    CU(cudaEventRecord(h->chunk_ev[C], h->copy_stream));
    h->chunk_b = C;
    *b_queued = true;
  }
  const double sh = h->opt.shift;
  ErrFlags *ep = h->d_err;
  auto prep = [&](int c) -> fastilu_status {  // gather + scale of chunk c
    CU(cudaStreamWaitEvent(st, h->chunk_ev[c], 0));
    CU(launch_tsell_gather_a_range(tdev(h), h->d_aval, rb(c), rb(c + 1), h->d_aT, st));
    const double *aT = h->d_aT;
    long long z0 = rb(c), z1 = rb(c + 1);
    double *sp = h->d_s, *adp = h->d_ad;
    void *args[] = {&aT, &z0, &z1, &sp, &adp, &ep, (void *)&sh};
    if (jit_launch(h->jit_scale, (int)((z1 - z0 + 255) / 256), 256, st, args)) FAIL(FASTILU_ERR_CUDA);
    return dbg("prep", c, 0);
  };
  auto ahat = [&](int c) -> fastilu_status {
    if (regp) {  // Â and iterate 0 of chunk c (its neighbours' scales exist now)
      CU(launch_tsell_init(tdev(h), h->d_aT, h->d_s, h->d_ad, rb(c), rb(c + 1), h->d_ahat,
                           h->d_vals[0], h->d_ud[0], h->d_err, sh, st, true));
      return dbg("init", c, 0);
    }
    const double *aT = h->d_aT, *sv = h->d_s;
    const unsigned long long *mk = h->d_tmask;
    long long z0 = rb(c), z1 = rb(c + 1);
    double *hp = h->d_ahat;
    long long zown = 0;
    void *args[] = {&aT, &sv, &mk, &z0, &z1, &hp, &ep, (void *)&sh, &zown};
    if (jit_launch(h->jit_ahat, (int)((z1 - z0 + 255) / 256), 256, st, args)) FAIL(FASTILU_ERR_CUDA);
    return dbg("ahat", c, 0);
  };
  int bufi[4] = {0, 1, 0, 1};  // ping-pong: iterate s in buffer s & 1
  if (nodiag && nsweeps == 2) bufi[1] = 1, bufi[2] = 0;
  if (nodiag && nsweeps == 3) bufi[1] = 2, bufi[2] = 0, bufi[3] = 1;
  auto vbuf = [&](int b) { return b == 2 ? h->d_vals3 : h->d_vals[b]; };
  auto ubuf = [&](int b) { return b == 2 ? h->d_ud3 : h->d_ud[b]; };
  auto tmapb = [&](int b) { return b == 2 ? h->st_tmap3.b : h->st_tmap[b].b; };
  auto tmapo = [&](int b) { return b == 2 ? h->st_tmap_own3.b : h->st_tmap_own[b].b; };
  auto sweep = [&](int sw, int c) -> fastilu_status {
    if (regp) {  // iterate s - 1 in d_vals[(s-1) & 1] (iterate 0 from the init kernel)
      const int ib = (sw - 1) & 1, ob = sw & 1;
      const double *old = h->d_vals[ib], *ahp = h->d_ahat, *udo = h->d_ud[ib];
      double *outp = h->d_vals[ob], *udn = h->d_ud[ob], *part = h->d_partials;
      const unsigned long long *mk = h->d_tmask;
      long long a0 = rb(c), a1 = rb(c + 1);
      double om = 1.0;
      unsigned long long *zp = &h->d_err->zero_pivot;
      unsigned int *ctr = h->d_counter;
      int sstr = h->t_sstride;
      const int64_t spt = h->t_rows_tile / 32, ss = h->t_sstride;
      const int64_t ntl = ((a1 - a0 + 31) / 32 + spt * ss - 1) / (spt * ss) * ss;
      void *fn = (sw == 1 && h->jit_sweep_first) ? h->jit_sweep_first : h->jit_sweep;
      void *args[] = {&old, &outp, &ahp, &mk, &udo, &udn, &a0, &a1, &om, &part, &zp, &ctr, &sstr};
      if (jit_launch(fn, (int)std::min<int64_t>(h->t_grid, ntl), h->t_threads, st, args))
        FAIL(FASTILU_ERR_CUDA);
      CU(launch_reduce_reset(h->d_partials, (int)ntl,
                             h->d_r2c + (int64_t)c * nsweeps + (sw - 1), h->d_counter, st));
      return dbg("sweep", sw, c);
    }
    const int ib = sw >= 2 ? bufi[sw - 1] : 0, ob = bufi[sw];
    const double *old = vbuf(ib), *ahp = h->d_ahat;
    double *outp = vbuf(ob), *udn = ubuf(ob), *part = h->d_partials;
    const unsigned long long *mk = h->d_tmask;
    long long a0 = rb(c), a1 = rb(c + 1);
    double om = 1.0;
    unsigned long long *zp = &h->d_err->zero_pivot;
    unsigned int *ctr = h->d_counter;
    void *sargs[] = {&old, &outp, &ahp, &mk, &udn, &a0, &a1, &om, &part, &zp, &ctr,
                     tmapb(ib), tmapo(ib)};
    void *fn = h->jit_st;
    int smem = h->st.smem, thr = h->st.threads, gmax = h->st_grid;
    int64_t Rk = R;
    if (sw == 1) {
      fn = h->jit_st_init;
      smem = h->st_init.smem;
      thr = h->st_init.threads;
      gmax = h->st_init_grid;
      Rk = h->st_init.rows;
      sargs[11] = h->st_tmap_ahat.b;
      sargs[12] = h->st_tmap_own_ahat.b;
    }
    const int64_t nt = (a1 - a0 + Rk - 1) / Rk;
    const int grid = (int)std::min<int64_t>(gmax, nt);
    if (jit_launch_smem(fn, grid, thr, smem, st, sargs)) FAIL(FASTILU_ERR_CUDA);
    CU(launch_reduce_reset(h->d_partials, (int)nt, h->d_r2c + (int64_t)c * nsweeps + (sw - 1),
                           h->d_counter, st));
    return dbg("sweep", sw, c);
  };
  auto diag = [&](int d) -> fastilu_status {  // step d: sweep s on chunk d - s + 1
    for (int sw = 1; sw <= nsweeps; sw++) {
      const int c = nodiag ? d : d - sw + 1;  // nodiag: all sweeps of chunk d
      if (c < 0 || c >= C) continue;
      fastilu_status fs = sweep(sw, c);
      if (fs) return fs;
    }
    return FASTILU_OK;
  };
  // apply pipeline (pipe_x), one buffer per Jacobi iterate (z^1..z^ntri, w^1..w^ntri: 2 ntri
  // vectors, 1.3 GB at c4) so that no iterate a later chunk still reads is overwritten:
  //  * L of chunk k, as soon as its factors are final: z^1 .. z^ntri of chunk k in turn (sweep t
  //    of chunk k reads z^{t-1} of chunks k-1 and k, both complete);
  //  * then the U cone: w^1 of chunk k, w^2 of chunk k-1, ..., w^ntri of chunk k-ntri+1 (sweep t
  //    of chunk c reads w^{t-1} of chunks c and c+1, and w^t of chunk c needs z of chunks
  //    c..c+t-1 only), so chunk c's x is final once chunk c + ntri - 1's z is, and goes back at
  //    once on its own stream (PCIe's other direction, concurrent with the upload).
  const double omt = h->opt.omega_tri;
  const int fb = nsweeps & 1;
  const double *fvals = h->d_vals[fb], *fud = h->d_ud[fb];
  double *xd = h->d_bx + h->n;
  if (pipe_x && !h->d2h_stream)
    CU(cudaStreamCreateWithFlags(&h->d2h_stream, cudaStreamNonBlocking));
  auto zt = [&](int t) { return h->d_it + (int64_t)(t - 1) * h->n; };           // z^t
  auto wt = [&](int t) { return h->d_it + (int64_t)(ntri + t - 1) * h->n; };    // w^t
  auto usweep = [&](int t, int c) -> fastilu_status {  // w^t of chunk c (+ x when t == ntri)
    if (t == 1)
      CU(launch_trisolve_first_U(zt(ntri), fud, h->d_s, wt(1), xd, rb(c), rb(c + 1), 0, omt,
                                 ntri == 1, st));
    else if (jit_jacobi(h, false, fvals, fud, zt(ntri), wt(t - 1), wt(t), xd, rb(c), rb(c + 1), 0,
                        omt, t == ntri))
      FAIL(FASTILU_ERR_CUDA);
    if (fastilu_status ds = dbg("usweep", t, c)) return ds;
    if (t == ntri) {  // x of chunk c is final
      CU(cudaEventRecord(h->x_ev[c], st));
      CU(cudaStreamWaitEvent(h->d2h_stream, h->x_ev[c], 0));
      CU(cudaMemcpyAsync(x_host + rb(c), xd + rb(c), sizeof(double) * (rb(c + 1) - rb(c)),
                         cudaMemcpyDeviceToHost, h->d2h_stream));
    }
    return FASTILU_OK;
  };
  // chunk k's factors are final (k = C .. C + ntri - 2: only the rest of the U cone)
  auto lu_chunk = [&](int k) -> fastilu_status {
    if (k < C) {
      CU(launch_trisolve_first_L(h->d_bx, h->d_s, h->d_y, zt(1), rb(k), rb(k + 1), 0, omt, st));
      for (int t = 2; t <= ntri; t++)
        if (jit_jacobi(h, true, fvals, nullptr, h->d_y, zt(t - 1), zt(t), nullptr, rb(k),
                       rb(k + 1), 0, omt, false))
          FAIL(FASTILU_ERR_CUDA);
      if (fastilu_status ds = dbg("L", k, 0)) return ds;
    }
    for (int t = 1; t <= ntri; t++) {
      const int c = k - t + 1;
      if (c < 0 || c >= C) continue;
      fastilu_status us = usweep(t, c);
      if (us) return us;
    }
    return FASTILU_OK;
  };
  fastilu_status fs;
  for (int c = 0; c < C; c++) {
    if ((fs = prep(c))) return fs;
    if (c >= 1) {
      if ((fs = ahat(c - 1))) return fs;
      if ((fs = diag(c - 1))) return fs;
      const int k = nodiag ? c - 1 : c - nsweeps;  // chunk whose factors are now final
      if (pipe_x && k >= 0 && (fs = lu_chunk(k))) return fs;
    }
  }
  if ((fs = ahat(C - 1))) return fs;
  for (int d = C - 1; d <= C + nsweeps - 2; d++) {
    if ((fs = diag(d))) return fs;
    const int k = nodiag ? d : d - nsweeps + 1;
    if (pipe_x && k >= 0 && k < C && (fs = lu_chunk(k))) return fs;
  }
  if (pipe_x) {
    CU(cudaEventRecord(h->ev[3], st));  // trace: factors and L sweeps done
    for (int k = C; k <= C + ntri - 2; k++)
      if ((fs = lu_chunk(k))) return fs;
  }
  CU(cudaEventRecord(h->ev[2], st));
  std::vector<double> r2c((size_t)C * nsweeps);
  CU(cudaMemcpyAsync(h->h_err, h->d_err, sizeof(ErrFlags), cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(r2c.data(), h->d_r2c, sizeof(double) * r2c.size(), cudaMemcpyDeviceToHost,
                     st));
  CU(cudaStreamSynchronize(st));
  if (pipe_x) {
    if (std::getenv("FASTILU_TRACE")) {  // timeline (ms from the compute's start)
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      CU(cudaEventRecord(e, h->d2h_stream));
      CU(cudaStreamSynchronize(h->d2h_stream));
      float t;
      std::fprintf(stderr, "fastilu trace (pipelined apply): chunks landed at");
      for (int c = 0; c < C; c++)
        if (cudaEventElapsedTime(&t, h->ev[0], h->chunk_ev[c]) == cudaSuccess)
          std::fprintf(stderr, " %.2f", t);
      if (cudaEventElapsedTime(&t, h->ev[0], h->ev[3]) == cudaSuccess)
        std::fprintf(stderr, "; factors+L_end %.2f", t);
      if (cudaEventElapsedTime(&t, h->ev[0], h->ev[2]) == cudaSuccess)
        std::fprintf(stderr, "; compute+apply_end %.2f", t);
      if (cudaEventElapsedTime(&t, h->ev[0], e) == cudaSuccess)
        std::fprintf(stderr, "; d2h_end %.2f", t);
      std::fprintf(stderr, " ms\n");
      cudaEventDestroy(e);
    }
    CU(cudaStreamSynchronize(h->copy_stream));
    CU(cudaStreamSynchronize(h->d2h_stream));
    *x_done = true;
  }
  h->have_values = true;
  h->t_init = 0.f;
  CU(cudaEventElapsedTime(&h->t_sweeps, h->ev[0], h->ev[2]));
  h->t_sweep1 = h->t_sweeps;
  h->last_ns = 0;
  h->resid.assign(nsweeps, 0.0);
  for (int sw = 0; sw < nsweeps; sw++) {
    double t = 0.0;
    for (int c = 0; c < C; c++) t += r2c[(size_t)c * nsweeps + sw];
    h->resid[sw] = std::sqrt(t);
  }
  h->cur = nsweeps & 1;
  h->vals_cur = h->d_vals[h->cur];
  h->ud_cur = h->d_ud[h->cur];
  ErrFlags ef = *h->h_err;
  if (ef.zero_diag != ~0ull) {
    h->err_index = (int64_t)ef.zero_diag + h->lbase;
    return FASTILU_ERR_ZERO_DIAG;
  }
  if (ef.zero_pivot != ~0ull) {
    h->err_index = (int64_t)ef.zero_pivot + h->lbase;
    return FASTILU_ERR_ZERO_PIVOT;
  }
  h->computed = true;
  return FASTILU_OK;
}

// On any failure after copies were queued, wait for the copy stream so that no DMA still reads
// the caller's buffers when the call returns (the caller may free them).
static fastilu_status drain_copies(fastilu_handle h, fastilu_status s) {
  if (s != FASTILU_OK && h->copy_stream) cudaStreamSynchronize(h->copy_stream);
  if (s != FASTILU_OK && h->d2h_stream) cudaStreamSynchronize(h->d2h_stream);
  return s;
}

extern "C" fastilu_status fastilu_compute_host(fastilu_handle h, const double *values,
                                               int nsweeps) {
  if (!h || !values || !h->d_aval || nsweeps < 0) FAIL(FASTILU_ERR_INVALID_ARG);
  DeviceGuard dg_(h->device);
  return drain_copies(h, compute_host_impl(h, values, nsweeps));
}

// fastilu_solve_host: compute_host(values, nsweeps) + apply_host(b, x, ntri), b's upload queued
// behind the values so that it lands during the compute's tail
extern "C" fastilu_status fastilu_solve_host(fastilu_handle h, const double *values, int nsweeps,
                                             const double *b, double *x, int ntrisweeps) {
  if (!h || !values || !h->d_aval || nsweeps < 0 || ntrisweeps < 1 ||
      (h->n > 0 && (!b || !x)))
    FAIL(FASTILU_ERR_INVALID_ARG);
  DeviceGuard dg_(h->device);
  bool queued = false, xdone = false;
  const bool pipe = std::getenv("FASTILU_SOLVE_NOPIPE") == nullptr;  // A/B: apply after compute
  fastilu_status s = drain_copies(
      h, compute_host_impl(h, values, nsweeps, b, &queued, pipe ? x : nullptr, ntrisweeps, &xdone));
  if (s) return s;
  if (xdone) {
    h->apply_timed = false;
    return FASTILU_OK;
  }
  if (!queued) return fastilu_apply_host(h, b, x, ntrisweeps);
  CU(cudaStreamWaitEvent(h->stream, h->chunk_ev[h->chunk_b], 0));
  CU(cudaEventRecord(h->ev[3], h->stream));
  s = apply_impl(h, h->d_bx, h->d_bx + h->n, ntrisweeps);
  if (s) return s;
  CU(cudaEventRecord(h->ev[4], h->stream));
  h->apply_timed = true;
  CU(cudaMemcpyAsync(x, h->d_bx + h->n, sizeof(double) * h->n, cudaMemcpyDeviceToHost,
                     h->stream));
  if (std::getenv("FASTILU_TRACE")) {  // timeline of the step (ms from the compute's start)
    cudaEvent_t e;
    CU(cudaEventCreate(&e));
    CU(cudaEventRecord(e, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    float t;
    std::fprintf(stderr, "fastilu trace: chunks landed at");
    for (int c = 0; c <= h->chunk_b; c++)
      if (cudaEventElapsedTime(&t, h->ev[0], h->chunk_ev[c]) == cudaSuccess)
        std::fprintf(stderr, " %.2f", t);
    cudaEvent_t marks[] = {h->ev[2], h->ev[3], h->ev[4], e};
    const char *names[] = {"compute_end", "apply_start", "apply_end", "d2h_end"};
    for (int q = 0; q < 4; q++)
      if (cudaEventElapsedTime(&t, h->ev[0], marks[q]) == cudaSuccess)
        std::fprintf(stderr, "; %s %.2f", names[q], t);
    std::fprintf(stderr, " ms\n");
    cudaEventDestroy(e);
  }
  CU(cudaStreamSynchronize(h->stream));
  return FASTILU_OK;
}

extern "C" fastilu_status fastilu_compute(fastilu_handle h, int nsweeps) {
  return compute_impl(h, nsweeps, 0.0, nullptr);
}

extern "C" fastilu_status fastilu_compute_async_block(fastilu_handle h, int nsweeps,
                                                      int nnz_per_thread) {
  if (!h || nnz_per_thread < 0) FAIL(FASTILU_ERR_INVALID_ARG);
  h->async_ept = nnz_per_thread;
  return compute_impl(h, nsweeps, 0.0, nullptr, false, true);
}

extern "C" fastilu_status fastilu_compute_async(fastilu_handle h, int nsweeps) {
  if (!h) FAIL(FASTILU_ERR_INVALID_ARG);
  h->async_ept = 0;  // default block size
  return compute_impl(h, nsweeps, 0.0, nullptr, false, true);
}

extern "C" fastilu_status fastilu_compute_warmup(fastilu_handle h, int nsweeps) {
  return compute_impl(h, nsweeps, 0.0, nullptr, true);
}

extern "C" fastilu_status fastilu_compute_tol(fastilu_handle h, double rtol, int max_sweeps,
                                              int *sweeps_done) {
  if (!(rtol > 0.0) || max_sweeps < 1) FAIL(FASTILU_ERR_INVALID_ARG);
  return compute_impl(h, max_sweeps, rtol, sweeps_done);
}

// --------------------------------------------------------------------------- apply
// one template-specialised Jacobi sweep (tsell.h jacobi_source); nonzero on a launch error
static int jit_jacobi(fastilu_handle h, bool lower, const double *vals, const double *ud,
                      const double *rhs, const double *xo, double *xn, double *xf, int64_t r0,
                      int64_t r1, int64_t Gh, double om, bool final_x) {
  if (r1 <= r0) return 0;
  const unsigned long long *mk = h->d_tmask;
  const double *sv = h->d_s;
  long long a0 = r0, a1 = r1, g = Gh;
  int fx = final_x ? 1 : 0;
  void *args[] = {&vals, &ud, &mk, &rhs, &xo, &xn, &xf, &sv, &a0, &a1, &g, &om, &fx};
  return jit_launch(h->jit_jac[lower ? 0 : 1], (int)((r1 - r0 + 255) / 256), 256, h->stream,
                    args);
}

static fastilu_status apply_impl(fastilu_handle h, const double *b, double *x, int ntri) {
  cudaStream_t st = h->stream;
  DevPattern P{h->d_rp, h->d_ci, h->d_dloc};
  const int64_t r0 = h->G, r1 = h->G + h->n;
  const double om = h->opt.omega_tri;
  const double *vals = h->vals_cur;
  const double *ud = h->ud_cur;
  if (ntri == 1) {  // one sweep each: x = s o (w (w y) / u_ii), one pass (no halo needed)
    CU(launch_trisolve_first_LU(b, h->d_s, ud, x, r0, r1, h->G, om, st));
    return FASTILU_OK;
  }
  // a8: L sweeps.  t = 1: z1 = w y with y = s o b (z0 = 0)
  CU(launch_trisolve_first_L(b, h->d_s, h->d_y, h->d_z[0], r0, r1, h->G, om, st));
  // multi-GPU template path: the vector halo of a sweep flies on the comm's halo stream while
  // the rows that read no ghost entry are swept (L: the first -o_0 owned rows read the lower
  // ghosts; U: the last o_{W-1} read the upper ones)
  const bool ovl = h->comm && h->tsell && h->jit_jac[0] && h->jit_jac[1] &&
                   !std::getenv("FASTILU_NO_HALO_OVERLAP");
  if (ovl) {
    const int64_t bl = std::min<int64_t>(h->n, -(int64_t)h->T.off[0]);
    const int64_t bu = std::min<int64_t>(h->n, (int64_t)h->T.off[h->T.W - 1]);
    for (int t = 2; t <= ntri; t++) {
      const double *zo = h->d_z[(t - 2) & 1];
      double *zn = h->d_z[(t - 1) & 1];
      cudaEvent_t done = nullptr;
      fastilu_status cs =
          comm_vector_halo_async(h->comm, h->d_z[(t - 2) & 1], st, true, false, &done);
      if (cs) return cs;
      if (jit_jacobi(h, true, vals, nullptr, h->d_y, zo, zn, nullptr, r0 + bl, r1, 0, om, false))
        FAIL(FASTILU_ERR_CUDA);
      CU(cudaStreamWaitEvent(st, done, 0));
      if (jit_jacobi(h, true, vals, nullptr, h->d_y, zo, zn, nullptr, r0, r0 + bl, 0, om, false))
        FAIL(FASTILU_ERR_CUDA);
    }
    const double *zf = h->d_z[(ntri - 1) & 1];
    CU(launch_trisolve_first_U(zf, ud, h->d_s, h->d_w[0], x, r0, r1, h->G, om, ntri == 1, st));
    for (int t = 2; t <= ntri; t++) {
      const double *wo = h->d_w[(t - 2) & 1];
      double *wn = h->d_w[(t - 1) & 1];
      cudaEvent_t done = nullptr;
      fastilu_status cs =
          comm_vector_halo_async(h->comm, h->d_w[(t - 2) & 1], st, false, true, &done);
      if (cs) return cs;
      if (jit_jacobi(h, false, vals, ud, zf, wo, wn, x, r0, r1 - bu, h->G, om, t == ntri))
        FAIL(FASTILU_ERR_CUDA);
      CU(cudaStreamWaitEvent(st, done, 0));
      if (jit_jacobi(h, false, vals, ud, zf, wo, wn, x, r1 - bu, r1, h->G, om, t == ntri))
        FAIL(FASTILU_ERR_CUDA);
    }
    return FASTILU_OK;
  }
  for (int t = 2; t <= ntri; t++) {
    const double *zo = h->d_z[(t - 2) & 1];
    if (h->comm) {
      fastilu_status cs = comm_vector_halo(h->comm, h->d_z[(t - 2) & 1], st, true, false);
      if (cs) return cs;
    }
    if (h->tsell && h->jit_jac[0]) {
      if (jit_jacobi(h, true, vals, nullptr, h->d_y, zo, h->d_z[(t - 1) & 1], nullptr, r0, r1,
                     0, om, false))
        FAIL(FASTILU_ERR_CUDA);
    } else if (h->tsell)
      CU(launch_tsell_jacobi(tdev(h), true, vals, nullptr, h->d_y, zo, h->d_z[(t - 1) & 1],
                             nullptr, nullptr, r0, r1, 0, om, false, st));
    else
      CU(launch_jacobi_L(P, vals, h->d_y, zo, h->d_z[(t - 1) & 1], r0, r1, om, h->G_tri, st));
  }
  const double *zf = h->d_z[(ntri - 1) & 1];
  // a9: U sweeps.  t = 1: w1 = w z / u_ii; the last sweep writes x = s o w
  CU(launch_trisolve_first_U(zf, ud, h->d_s, h->d_w[0], x, r0, r1, h->G, om, ntri == 1, st));
  for (int t = 2; t <= ntri; t++) {
    if (h->comm) {
      fastilu_status cs = comm_vector_halo(h->comm, h->d_w[(t - 2) & 1], st, false, true);
      if (cs) return cs;
    }
    if (h->tsell && h->jit_jac[1]) {
      if (jit_jacobi(h, false, vals, ud, zf, h->d_w[(t - 2) & 1], h->d_w[(t - 1) & 1], x, r0, r1,
                     h->G, om, t == ntri))
        FAIL(FASTILU_ERR_CUDA);
    } else if (h->tsell)
      CU(launch_tsell_jacobi(tdev(h), false, vals, ud, zf, h->d_w[(t - 2) & 1],
                             h->d_w[(t - 1) & 1], x, h->d_s, r0, r1, h->G, om, t == ntri, st));
    else
      CU(launch_jacobi_U(P, vals, ud, zf, h->d_w[(t - 2) & 1], h->d_w[(t - 1) & 1], x, h->d_s,
                         r0, r1, h->G, om, t == ntri, h->G_tri, st));
  }
  return FASTILU_OK;
}

extern "C" fastilu_status fastilu_apply(fastilu_handle h, const double *b, double *x,
                                        int ntrisweeps) {
  if (!h || ntrisweeps < 1 || (h->n > 0 && (!b || !x))) FAIL(FASTILU_ERR_INVALID_ARG);
  if (!h->computed) FAIL(FASTILU_ERR_STATE);
  DeviceGuard dg_(h->device);
  (void)cudaGetLastError();  // clear a non-sticky error left by the caller's own CUDA work
  CU(cudaEventRecord(h->ev[3], h->stream));
  fastilu_status s = apply_impl(h, b, x, ntrisweeps);
  if (s) return s;
  CU(cudaEventRecord(h->ev[4], h->stream));
  h->apply_timed = true;
  return FASTILU_OK;
}

extern "C" fastilu_status fastilu_apply_host(fastilu_handle h, const double *b, double *x,
                                             int ntrisweeps) {
  if (!h || ntrisweeps < 1 || (h->n > 0 && (!b || !x))) FAIL(FASTILU_ERR_INVALID_ARG);
  if (!h->computed) FAIL(FASTILU_ERR_STATE);
  DeviceGuard dg_(h->device);
  (void)cudaGetLastError();  // clear a non-sticky error left by the caller's own CUDA work
  if (!h->d_bx) CU(dalloc(&h->d_bx, 2 * h->n));
  CU(cudaMemcpyAsync(h->d_bx, b, sizeof(double) * h->n, cudaMemcpyHostToDevice, h->stream));
  CU(cudaEventRecord(h->ev[3], h->stream));
  fastilu_status s = apply_impl(h, h->d_bx, h->d_bx + h->n, ntrisweeps);
  if (s) return s;
  CU(cudaEventRecord(h->ev[4], h->stream));
  h->apply_timed = true;
  CU(cudaMemcpyAsync(x, h->d_bx + h->n, sizeof(double) * h->n, cudaMemcpyDeviceToHost,
                     h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return FASTILU_OK;
}

// --------------------------------------------------------------------------- GMRES (config 5)
// Restarted GMRES(m) with right preconditioning x = M^-1 y, M^-1 = fastilu_apply (a fixed
// linear operator: ntri Jacobi sweeps from 0), classical Gram-Schmidt with the
// reorthogonalisation delayed by one step (DCGS2: one batched multi-dot pass and one update pass
// over V per iteration instead of m sequential MGS dots), Givens rotations on the host, x0 = 0,
// convergence on the relative residual ||b - A x|| / ||b|| <= rtol (
// SPEC.md:416-456).
extern "C" fastilu_status fastilu_gmres(fastilu_handle h, const double *b, double *x,
                                        int restart, double rtol, int max_iters,
                                        int ntrisweeps, int *iters_out, double *relres_out) {
  if (!h || restart < 1 || restart > 120 || !(rtol > 0.0) || max_iters < 1 || ntrisweeps < 1 ||
      (h->n > 0 && (!b || !x)))
    FAIL(FASTILU_ERR_INVALID_ARG);
  if (!h->computed) FAIL(FASTILU_ERR_STATE);
  DeviceGuard dg_(h->device);
  (void)cudaGetLastError();  // clear a non-sticky error left by the caller's own CUDA work
  cudaStream_t st = h->stream;
  const int64_t n = h->n;
  const int m = restart;
  if (h->gm_m < m) {
    void *old[] = {h->gm_V, h->gm_w, h->gm_ext, h->gm_u, h->gm_r, h->gm_part, h->gm_c};
    for (void *p : old)
      if (p) cudaFree(p);
    if (h->gm_hbuf) cudaFreeHost(h->gm_hbuf);
    CU(dalloc(&h->gm_V, (int64_t)(m + 1) * std::max<int64_t>(n, 1)));
    CU(dalloc(&h->gm_w, n));
    CU(dalloc(&h->gm_ext, h->E));
    CU(cudaMemset(h->gm_ext, 0, sizeof(double) * h->E));
    CU(dalloc(&h->gm_u, n));
    CU(dalloc(&h->gm_r, n));
    CU(dalloc(&h->gm_part, (int64_t)2 * (m + 3) * kDotBlocks));
    // dots (2 (m + 2)) | coefficients (2 (m + 2))
    CU(dalloc(&h->gm_c, 4 * (m + 2)));
    CU(cudaMallocHost((void **)&h->gm_hbuf, sizeof(double) * 4 * (m + 2)));
    h->gm_m = m;
  }
  double *V = h->gm_V, *w = h->gm_w, *u = h->gm_u, *r = h->gm_r;
  // test hook: re-project every pending vector explicitly once (the severe-cancellation branch)
  const bool force_reproject = std::getenv("FASTILU_GMRES_FORCE_REPROJECT") != nullptr;
  h->gm_reorth = 0;
  h->gm_retry = 0;
  const int64_t ldv = std::max<int64_t>(n, 1);
  // collective dot products: k local partial sums -> host -> sum over ranks
  auto dots = [&](int k, const double *vecs, const double *vec, double *out) -> fastilu_status {
    CU(launch_mdot(vecs, ldv, k, vec, n, h->gm_part, h->gm_c, st));
    CU(cudaMemcpyAsync(h->gm_hbuf, h->gm_c, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    for (int q = 0; q < k; q++) out[q] = h->gm_hbuf[q];
    if (h->comm) {
      ErrFlags dummy{~0ull, ~0ull};
      return comm_allreduce_host(h->comm, out, k, dummy);
    }
    return FASTILU_OK;
  };
  auto spmv = [&](const double *v, double *y) -> fastilu_status {  // y = A v
    CU(cudaMemcpyAsync(h->gm_ext + h->G, v, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    if (h->comm) {
      fastilu_status cs = comm_vector_halo(h->comm, h->gm_ext, st, true, true);
      if (cs) return cs;
    }
    if (h->tsell && h->jit_spmv) {
      const double *aT = h->d_aT, *xe = h->gm_ext;
      const unsigned long long *mk = h->d_tmask;
      long long a0 = h->G, a1 = h->G + n, gh = h->G;
      void *args[] = {&aT, &mk, &xe, &y, &a0, &a1, &gh};
      if (n > 0 && jit_launch(h->jit_spmv, (int)((n + 255) / 256), 256, st, args))
        FAIL(FASTILU_ERR_CUDA);
      return FASTILU_OK;
    }
    CU(launch_spmv(h->d_arp, h->d_aci, h->d_aval, h->gm_ext, y, h->G, h->G + n, h->G, h->G_spmv,
                   st));
    return FASTILU_OK;
  };
  auto nrm = [&](const double *v, double *out) -> fastilu_status {
    fastilu_status fs = dots(1, v, v, out);
    *out = std::sqrt(*out);
    return fs;
  };
  fastilu_status fs;
  CU(cudaEventRecord(h->ev[3], st));
  CU(cudaMemsetAsync(x, 0, sizeof(double) * n, st));
  CU(cudaMemcpyAsync(r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  double bnorm = 0.0;
  if ((fs = nrm(b, &bnorm))) return fs;
  double beta = bnorm;
  int total = 0;
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1);
  // Givens rotation of column j (rows 0..j+1 of Rm) with the previous rotations; new residual
  // estimate in g[j + 1]
  auto givens = [&](std::vector<double> &Rm, int j) {
    for (int q = 0; q < j; q++) {
      const double a = Rm[(size_t)q * m + j], c = Rm[(size_t)(q + 1) * m + j];
      Rm[(size_t)q * m + j] = cs[q] * a + sn[q] * c;
      Rm[(size_t)(q + 1) * m + j] = -sn[q] * a + cs[q] * c;
    }
    const double a = Rm[(size_t)j * m + j], c = Rm[(size_t)(j + 1) * m + j];
    const double rr = std::hypot(a, c);
    cs[j] = rr > 0.0 ? a / rr : 1.0;
    sn[j] = rr > 0.0 ? c / rr : 0.0;
    Rm[(size_t)j * m + j] = rr;
    Rm[(size_t)(j + 1) * m + j] = 0.0;
    g[j + 1] = -sn[j] * g[j];
    g[j] = cs[j] * g[j];
  };
  // x += M^-1 (V y), y = R^-1 g (upper triangular k x k); then r = b - A x, beta = ||r||
  auto finish_cycle = [&](const std::vector<double> &Rm, int k) -> fastilu_status {
    std::vector<double> y(k, 0.0);
    for (int q = k - 1; q >= 0; q--) {
      double t = g[q];
      for (int c2 = q + 1; c2 < k; c2++) t -= Rm[(size_t)q * m + c2] * y[c2];
      y[q] = t / Rm[(size_t)q * m + q];
    }
    for (int q = 0; q < k; q++) h->gm_hbuf[q] = y[q];
    CU(cudaMemcpyAsync(h->gm_c, h->gm_hbuf, sizeof(double) * k, cudaMemcpyHostToDevice, st));
    CU(cudaMemsetAsync(w, 0, sizeof(double) * n, st));
    CU(launch_maxpy(V, ldv, k, h->gm_c, w, n, 1.0, st));
    fastilu_status fs2 = apply_impl(h, w, u, ntrisweeps);
    if (fs2) return fs2;
    CU(launch_axpby(1.0, u, 1.0, x, n, st));
    if ((fs2 = spmv(x, w))) return fs2;
    CU(cudaMemcpyAsync(r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    CU(launch_axpby(-1.0, w, 1.0, r, n, st));
    return nrm(r, &beta);
  };
  // DCGS2 Arnoldi: V_p is the PENDING vector (projected once, not yet
  // normalised); step p applies B = A M^-1 to it, takes all dots V_j . V_p and V_j . (B V_p),
  // j <= p, in ONE pass and ONE synchronisation, which (i) finishes the reorthogonalisation of
  // V_p -- q_p = (V_p - Q s) / rho, rho^2 = ||V_p||^2 - ||s||^2 -- and with it Hessenberg column
  // p - 1 (H[:p, p-1] += s, H[p, p-1] = rho), and (ii) gives the first projection of B q_p
  // without applying B again: B q_p = (B V_p - B Q s) / rho with B Q = Q H, so
  // h_p = (c - H s) / rho and the next pending vector is (B V_p - Q_{p+1} c) / rho, c = [z,
  // (zeta - s.z) / rho].  A second pass over V does both updates.  The rotated copy R of H drives
  // the least-squares problem; the residual estimate of column p - 1 is known at step p.
  std::vector<double> R((size_t)(m + 1) * m), dv(2 * (m + 2)), sv(m + 1), zv(m + 1);
  while (bnorm > 0.0 && beta / bnorm > rtol && total < max_iters) {
    CU(cudaMemcpyAsync(V, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));  // pending V_0
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(R.begin(), R.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    int p = 0, k = 0, retries = 0;
    for (;;) {
      const bool last = p == m || (p >= 1 && total + 1 >= max_iters);
      if (!last) {
        if ((fs = apply_impl(h, V + p * ldv, u, ntrisweeps))) return fs;  // u = M^-1 V_p
        if ((fs = spmv(u, w))) return fs;                                   // w = A u
      }
      CU(launch_dcgs_dot(V, ldv, p, last ? nullptr : w, n, h->gm_part, h->gm_c, st));
      CU(cudaMemcpyAsync(h->gm_hbuf, h->gm_c, sizeof(double) * 2 * (p + 1),
                         cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
      for (int q = 0; q < 2 * (p + 1); q++) dv[q] = h->gm_hbuf[q];
      if (h->comm) {
        ErrFlags dummy{~0ull, ~0ull};
        if ((fs = comm_allreduce_host(h->comm, dv.data(), 2 * (p + 1), dummy))) return fs;
      }
      double ss = 0.0, sz = 0.0;
      for (int q = 0; q < p; q++) {
        sv[q] = dv[2 * q];
        zv[q] = dv[2 * q + 1];
        ss += sv[q] * sv[q];
        sz += sv[q] * zv[q];
      }
      const double alpha = dv[2 * p], zeta = dv[2 * p + 1], rho2 = alpha - ss;
      if (p >= 1 && alpha > 0.0 && (rho2 < 0.5 * alpha || (force_reproject && retries == 0)) &&
          retries < 2) {
        // the pending vector still leans on Q (severe cancellation in its first projection):
        // project it explicitly, fold s into column p - 1 and redo the step
        for (int q = 0; q < p; q++) {
          h->gm_hbuf[2 * (m + 2) + q] = sv[q];
          H[(size_t)q * m + p - 1] += sv[q];
        }
        CU(cudaMemcpyAsync(h->gm_c + 2 * (m + 2), h->gm_hbuf + 2 * (m + 2), sizeof(double) * p,
                           cudaMemcpyHostToDevice, st));
        CU(launch_maxpy(V, ldv, p, h->gm_c + 2 * (m + 2), V + p * ldv, n, -1.0, st));
        retries++;
        h->gm_retry++;
        continue;
      }
      retries = 0;
      const double rho = rho2 > 0.0 ? std::sqrt(rho2) : 0.0;
      if (p >= 1) {  // column p - 1 is final
        for (int q = 0; q < p; q++) H[(size_t)q * m + p - 1] += sv[q];
        H[(size_t)p * m + p - 1] = rho;
        for (int q = 0; q <= p; q++) R[(size_t)q * m + p - 1] = H[(size_t)q * m + p - 1];
        givens(R, p - 1);
        total++;
        h->gm_reorth++;
        k = p;
        if (last || rho == 0.0 || std::fabs(g[p]) <= rtol * bnorm) break;
      } else {
        g[0] = rho;  // ||r||
        if (rho == 0.0) break;
      }
      const double cp = (zeta - sz) / rho;
      for (int q = 0; q <= p; q++) {  // tentative column p: (c - H[0..p, 0..p-1] s) / rho
        double t = q < p ? zv[q] : cp;
        for (int l = std::max(0, q - 1); l < p; l++) t -= H[(size_t)q * m + l] * sv[l];
        H[(size_t)q * m + p] = t / rho;
      }
      double *cb = h->gm_hbuf + 2 * (m + 2);
      for (int q = 0; q < p; q++) {
        cb[q] = sv[q];
        cb[p + q] = zv[q];
      }
      cb[2 * p] = cp;
      cb[2 * p + 1] = 1.0 / rho;
      CU(cudaMemcpyAsync(h->gm_c + 2 * (m + 2), cb, sizeof(double) * (2 * p + 2),
                         cudaMemcpyHostToDevice, st));
      CU(launch_dcgs_update(V, ldv, p, h->gm_c + 2 * (m + 2), w, n, st));
      p++;
    }
    if ((fs = finish_cycle(R, k))) return fs;
  }
  CU(cudaEventRecord(h->ev[4], st));
  h->apply_timed = true;
  CU(cudaStreamSynchronize(st));
  if (iters_out) *iters_out = total;
  if (relres_out) *relres_out = bnorm > 0.0 ? beta / bnorm : 0.0;
  return FASTILU_OK;
}

// --------------------------------------------------------------------------- introspection
extern "C" fastilu_status fastilu_get_device(fastilu_handle h, int *device) {
  if (!h || !device) FAIL(FASTILU_ERR_INVALID_ARG);
  *device = h->device;
  return FASTILU_OK;
}

extern "C" fastilu_status fastilu_get_sizes(fastilu_handle h, int64_t *n, int64_t *nnz_S,
                                            int64_t *nnz_A) {
  if (!h) FAIL(FASTILU_ERR_INVALID_ARG);
  if (n) *n = h->n;
  if (nnz_S) *nnz_S = (int64_t)h->h_ci.size();
  if (nnz_A) {
    // A entries of the owned rows
    *nnz_A = h->nnzA_loc;
    if (h->G && h->d_arp) {
      int64_t g = 0;
      cudaMemcpy(&g, h->d_arp + h->G, sizeof(int64_t), cudaMemcpyDeviceToHost);
      *nnz_A -= g;
    }
  }
  return FASTILU_OK;
}

extern "C" fastilu_status fastilu_get_pattern(fastilu_handle h, int64_t *row_ptr,
                                              int32_t *col_idx, int8_t *level) {
  if (!h) FAIL(FASTILU_ERR_INVALID_ARG);
  if (row_ptr) std::memcpy(row_ptr, h->h_rp.data(), sizeof(int64_t) * h->h_rp.size());
  if (col_idx) std::memcpy(col_idx, h->h_ci.data(), sizeof(int32_t) * h->h_ci.size());
  if (level) std::memcpy(level, h->h_lev.data(), h->h_lev.size());
  return FASTILU_OK;
}

extern "C" fastilu_status fastilu_get_factors(fastilu_handle h, double *vals, double *s) {
  if (!h) FAIL(FASTILU_ERR_INVALID_ARG);
  if (!h->computed) FAIL(FASTILU_ERR_STATE);
  DeviceGuard dg_(h->device);
  (void)cudaGetLastError();  // clear a non-sticky error left by the caller's own CUDA work
  CU(cudaStreamSynchronize(h->stream));
  if (vals && h->tsell) {  // gather the owned rows' S entries out of the template slots
    const Template &T = h->T;
    std::vector<double> tv((size_t)h->nsl * T.W * 32);
    CU(cudaMemcpy(tv.data(), h->vals_cur, sizeof(double) * tv.size(), cudaMemcpyDeviceToHost));
    for (int64_t r = 0; r < h->n; r++) {
      const int64_t i = h->G + r, g = h->row_begin + r;
      for (int64_t p = h->h_rp[r]; p < h->h_rp[r + 1]; p++) {
        const int32_t o = (int32_t)(h->h_ci[p] - g);
        const int w = (int)(std::lower_bound(T.off.begin(), T.off.end(), o) - T.off.begin());
        vals[p] = tv[((i >> 5) * T.W + w) * 32 + (i & 31)];
      }
    }
  } else if (vals) {
    CU(cudaMemcpy(vals, h->vals_cur + h->own_off, sizeof(double) * h->nnz_own,
                  cudaMemcpyDeviceToHost));
  }
  if (s) CU(cudaMemcpy(s, h->d_s + h->G, sizeof(double) * h->n, cudaMemcpyDeviceToHost));
  return FASTILU_OK;
}

extern "C" fastilu_status fastilu_set_factors(fastilu_handle h, const double *vals,
                                              const double *s) {
  if (!h || (h->nnz_own > 0 && !vals) || (h->n > 0 && !s)) FAIL(FASTILU_ERR_INVALID_ARG);
  if (h->bsr && !h->d_vals[0]) FAIL(FASTILU_ERR_UNSUPPORTED);
  DeviceGuard dg_(h->device);
  (void)cudaGetLastError();
  CU(cudaStreamSynchronize(h->stream));
  h->computed = false;
  h->err_index = -1;
  // u_ii of the owned rows (local index G + r), zero-pivot check
  std::vector<double> ud((size_t)h->E, 0.0);
  for (int64_t r = 0; r < h->n; r++) {
    const int64_t g = h->row_begin + r;
    double d = 0.0;
    for (int64_t p = h->h_rp[r]; p < h->h_rp[r + 1]; p++)
      if (h->h_ci[p] == g) d = vals[p];
    if (!(d != 0.0 && std::fabs(d) <= 1.7976931348623157e308)) {
      h->err_index = g;
      return FASTILU_ERR_ZERO_PIVOT;
    }
    ud[(size_t)(h->G + r)] = d;
  }
  if (h->tsell) {  // scatter into the template slots (absent / ghost slots +0.0)
    const Template &T = h->T;
    std::vector<double> tv((size_t)h->nsl * T.W * 32, 0.0);
    for (int64_t r = 0; r < h->n; r++) {
      const int64_t i = h->G + r, g = h->row_begin + r;
      for (int64_t p = h->h_rp[r]; p < h->h_rp[r + 1]; p++) {
        const int32_t o = (int32_t)(h->h_ci[p] - g);
        const int w = (int)(std::lower_bound(T.off.begin(), T.off.end(), o) - T.off.begin());
        tv[((i >> 5) * T.W + w) * 32 + (i & 31)] = vals[p];
      }
    }
    CU(cudaMemcpy(h->d_vals[0], tv.data(), sizeof(double) * tv.size(), cudaMemcpyHostToDevice));
  } else {
    CU(cudaMemcpy(h->d_vals[0] + h->own_off, vals, sizeof(double) * h->nnz_own,
                  cudaMemcpyHostToDevice));
  }
  CU(cudaMemcpy(h->d_ud[0], ud.data(), sizeof(double) * ud.size(), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(h->d_s + h->G, s, sizeof(double) * h->n, cudaMemcpyHostToDevice));
  h->cur = 0;
  h->vals_cur = h->d_vals[0];
  h->ud_cur = h->d_ud[0];
  h->resid.clear();
  h->computed = true;
  return FASTILU_OK;
}

extern "C" fastilu_status fastilu_get_residual_history(fastilu_handle h, double *hist, int cap,
                                                       int *count) {
  if (!h) FAIL(FASTILU_ERR_INVALID_ARG);
  int c = std::min<int>(cap, (int)h->resid.size());
  for (int i = 0; i < c; i++) hist[i] = h->resid[i];
  if (count) *count = c;
  return FASTILU_OK;
}

extern "C" fastilu_status fastilu_get_timings(fastilu_handle h, double *t3) {
  if (!h || !t3) FAIL(FASTILU_ERR_INVALID_ARG);
  DeviceGuard dg_(h->device);
  float ta = 0.f;
  if (h->apply_timed && cudaEventQuery(h->ev[4]) == cudaSuccess &&
      cudaEventElapsedTime(&ta, h->ev[3], h->ev[4]) != cudaSuccess) {
    (void)cudaGetLastError();  // never leave a non-sticky error behind for the next launch check
    ta = 0.f;
  }
  t3[0] = h->t_init;
  t3[1] = h->t_sweeps;
  t3[2] = ta;
  return FASTILU_OK;
}

extern "C" fastilu_status fastilu_get_sweep_split(fastilu_handle h, double *t2) {
  if (!h || !t2) FAIL(FASTILU_ERR_INVALID_ARG);
  t2[0] = h->t_sweep1;
  t2[1] = h->last_ns >= 2 ? (double)h->t_sweeps - (double)h->t_sweep1 : 0.0;
  return FASTILU_OK;
}

extern "C" fastilu_status fastilu_get_info(fastilu_handle h, char *buf, int cap) {
  if (!h || !buf || cap < 1) FAIL(FASTILU_ERR_INVALID_ARG);
  char tmp[1024];
  if (h->tsell)
    snprintf(tmp, sizeof(tmp),
             "path=tsell W=%d c0=%d WA=%d terms=%zu threads=%d rows/tile=%d grid=%d regs=%d "
             "local=%d tiles=%lld sstride=%d G=%lld H=%lld",
             h->T.W, h->T.c0, h->T.WA, h->T.terms.size(), h->t_threads, h->t_rows_tile,
             h->t_grid, h->t_regs,
             h->t_spill, (long long)h->t_ntiles, h->t_sstride, (long long)h->G, (long long)h->H);
  if (h->tsell && h->jit_st) {
    const size_t L = strlen(tmp);
    snprintf(tmp + L, sizeof(tmp) - L,
             " staged=1 st_threads=%d st_parts=%d st_rows=%d st_shift=%d st_groups=%d "
             "st_box=32x%dx%d st_stages=%d st_smem_kb=%d st_grid=%d st_init=%d "
             "st_init_parts=%d st_init_rows=%d st_lds=%d st_tma=%lld st_init_lds=%d "
             "st_init_tma=%lld st_opts=%u st_init_opts=%u",
             h->st.threads, h->st.parts, h->st.rows, h->st.shift, h->st.ngroups, h->st.box_cols,
             h->st.box_slices, h->st.stages, h->st.smem / 1024, h->st_grid,
             h->jit_st_init ? 1 : 0, h->st_init.parts, h->st_init.rows, h->st.lds_per_row,
             h->st.tma_bytes_per_tile, h->jit_st_init ? h->st_init.lds_per_row : 0,
             h->jit_st_init ? h->st_init.tma_bytes_per_tile : 0LL, h->st.opts,
             h->jit_st_init ? h->st_init.opts : 0u);
  }
  if (h->tsell) {
  } else if (h->bsr)
    snprintf(tmp, sizeof(tmp),
             "path=bsr%d blocks=%lld terms=%lld threads=%d grid=%d smem_kb=%d minb=%d "
             "tri_lanes=%d G=%lld H=%lld",
             h->B.bs, (long long)h->B.nblk, (long long)h->bsr_nterms,
             h->bsr_threads, h->bsr_grid, (int)(h->bsr_smem / 1024), h->bsr_minb, h->G_tri, (long long)h->G, (long long)h->H);
  else
    snprintf(tmp, sizeof(tmp),
             "path=%s G_lanes=%d E=%d threads=%d grid=%d classes=%lld tri_lanes=%d G=%lld H=%lld",
             h->scfg.prog ? "csr-classes" : (h->scfg.hash ? "csr-hash" : "csr-bsearch"),
             h->scfg.G, h->scfg.E, h->scfg.threads, h->scfg.grid, (long long)h->nclasses,
             h->G_tri, (long long)h->G, (long long)h->H);
  if (h->comm) {  // multi-GPU: ranks and the bytes this rank sends per factor halo
    const size_t L = strlen(tmp);
    snprintf(tmp + L, sizeof(tmp) - L, " nranks=%d halo_bytes=%lld", h->opt.nranks,
             (long long)comm_halo_bytes(h->comm, h->tsell ? h->T.W : 0, h->tsell ? h->T.c0 : 0));
  }
  {
    const size_t L = strlen(tmp);
    snprintf(tmp + L, sizeof(tmp) - L, " gmres_reorth=%d gmres_retry=%d", h->gm_reorth,
             h->gm_retry);
  }
  snprintf(buf, cap, "%s", tmp);
  return FASTILU_OK;
}

extern "C" fastilu_status fastilu_destroy(fastilu_handle h) {
  if (!h) return FASTILU_OK;
  DeviceGuard dg_(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->comm) comm_destroy(h->comm);
  void *ptrs[] = {h->d_rp,    h->d_ci,    h->d_dloc,     h->d_arp,  h->d_aci,     h->d_apos,
                  h->d_adiag, h->d_aval,  h->d_vals[0],  h->d_vals[1], h->d_ud[0], h->d_ud[1],
                  h->d_ahat,  h->d_s,     h->d_ad,       h->d_y,    h->d_z[0],    h->d_z[1],
                  h->d_w[0],  h->d_w[1],  h->d_bx,       h->d_partials, h->d_r2,  h->d_err,
                  h->d_rclass, h->d_coff, h->d_caoff, h->d_prog, h->d_toff, h->d_toffA,
                  h->d_tasrc, h->d_tw2a, h->d_tmask, h->d_counter, h->gm_V, h->gm_w,
                  h->gm_ext, h->gm_u, h->gm_r, h->gm_part, h->gm_c, h->d_aT,
                  h->d_bptr, h->d_tptr, h->d_brow, h->d_bcol, h->d_bdiag, h->d_terms,
                  h->d_vb[0], h->d_vb[1], h->d_ahb};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  if (h->h_err) cudaFreeHost(h->h_err);
  if (h->h_r2) cudaFreeHost(h->h_r2);
  if (h->gm_hbuf) cudaFreeHost(h->gm_hbuf);
  for (auto *p : h->d_lmask) cudaFree(p);
  for (int i = 0; i < 6; i++)
    if (h->ev[i]) cudaEventDestroy(h->ev[i]);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  for (cudaEvent_t e : h->chunk_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : h->x_ev) cudaEventDestroy(e);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  if (h->d2h_stream) cudaStreamDestroy(h->d2h_stream);
  if (h->d_it) cudaFree(h->d_it);
  if (h->d_vals3) cudaFree(h->d_vals3);
  if (h->d_ud3) cudaFree(h->d_ud3);
  if (h->d_r2c) cudaFree(h->d_r2c);
  delete h;
  return FASTILU_OK;
}
