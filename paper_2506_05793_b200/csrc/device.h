// Private device-side launch interface of libfastilu_b200 (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace fastilu {

// Local layout: rows of S are stored row-major in one CSR
// (strict-lower part = L without its unit diagonal, then the diagonal, then the strict upper
// part of U), local row r <-> global row lbase + r.  Local rows [0, G) are ghost rows of the
// lower neighbour (multi-GPU only), [G, G + n) are owned.  Column indices are LOCAL
// (global - lbase); vectors are extended [G ghost | n owned | H upper ghost].
struct DevPattern {
  const int64_t *rp;    // nloc + 1
  const int32_t *ci;    // nnz_loc, local columns
  const int32_t *dloc;  // nloc: offset of the diagonal inside the row (= #L entries)
};

struct SweepCfg {
  int G;            // lanes per row group (4, 8, 16, 32)
  int threads;      // threads per block
  int cap_m;        // smem capacity for the row's entries
  bool hash;        // injective offset hash available (else binary search)
  uint32_t hmul;    // hash: slot = ((j - i) * hmul) >> hshift
  int hshift;
  int hsize;        // table entries (power of two)
  int grid;         // blocks (= resident capacity)
  int64_t chunk;    // rows per block
  size_t smem;      // dynamic smem per block
  bool prog;        // class-program kernel (else hash / binary-search kernel)
  int E;            // prog kernel: U-row entries per lane per pivot (1, 2, 4)
};

struct ProgView {
  const int32_t *row_class;  // per owned row
  const int64_t *class_off;  // program byte offset per class
  const int32_t *class_aoff; // A-position part offset per class
  const uint8_t *prog;
};

struct ErrFlags;

struct SweepArgs {
  DevPattern P;
  const int64_t *arp;     // A row pointers (local rows)
  const int32_t *apos;    // offset of each A entry inside its S row
  const double *ahatA;    // ahat on A's pattern
  const double *old;      // iterate s-1 (S layout)
  double *out;            // iterate s
  const double *udo;      // u_ii of iterate s-1
  double *udn;            // u_ii of iterate s
  int64_t r0, r1;         // local rows to sweep
  double omega;
  double *partials;       // per-block residual partials
  ErrFlags *err;
};

struct ErrFlags {
  unsigned long long zero_diag;   // min local row with a_ii == 0
  unsigned long long zero_pivot;  // min local row with u_ii == 0 / non-finite in an iterate
};

// Manteuffel shift: a_ii' = a_ii + shift |a_ii| (shift = 0: unchanged, bitwise)
cudaError_t launch_scale(const int64_t *arp, const int32_t *adiag, const double *aval,
                         int64_t r0, int64_t r1, double *s, double *ad, ErrFlags *err,
                         double shift, cudaStream_t st);

cudaError_t launch_init(const DevPattern &P, const int64_t *arp, const int32_t *aci,
                        const int32_t *apos, const double *aval, const double *s,
                        const double *ad, int64_t r0, int64_t r1, double *ahatA, double *vals,
                        double *udiag, ErrFlags *err, int G, double shift, cudaStream_t st);

// sets the smem attribute and returns the resident blocks per SM for cfg
cudaError_t sweep_configure(const SweepCfg &cfg, int *blocks_per_sm);
cudaError_t launch_sweep(const SweepArgs &a, const SweepCfg &cfg, cudaStream_t st);
cudaError_t sweep_prog_configure(const SweepCfg &cfg, int *blocks_per_sm);
cudaError_t launch_sweep_prog(const SweepArgs &a, const ProgView &pv, const SweepCfg &cfg,
                              cudaStream_t st);

cudaError_t launch_reduce(const double *partials, int np, double *dst, cudaStream_t st);

// y = s o b (b indexed by owned row), z1 = omega * y
cudaError_t launch_trisolve_first_L(const double *b, const double *s, double *y, double *z,
                                    int64_t r0, int64_t r1, int64_t G, double omega,
                                    cudaStream_t st);
// w1 = omega * z / u_ii; if final: x[r - G] = s * w1
// ntri = 1 in one pass: x[r - G] = s o (omega (omega (s o b)) / u_ii), bitwise first_L + first_U
cudaError_t launch_trisolve_first_LU(const double *b, const double *s, const double *udiag,
                                     double *x, int64_t r0, int64_t r1, int64_t G, double omega,
                                     cudaStream_t st);
cudaError_t launch_trisolve_first_U(const double *z, const double *udiag, const double *s,
                                    double *w, double *x, int64_t r0, int64_t r1, int64_t G,
                                    double omega, bool final, cudaStream_t st);
cudaError_t launch_jacobi_L(const DevPattern &P, const double *vals, const double *y,
                            const double *zold, double *znew, int64_t r0, int64_t r1,
                            double omega, int G, cudaStream_t st);
cudaError_t launch_jacobi_U(const DevPattern &P, const double *vals, const double *udiag,
                            const double *z, const double *wold, double *wnew, double *x,
                            const double *s, int64_t r0, int64_t r1, int64_t Gh, double omega,
                            bool final, int G, cudaStream_t st);

// ---- template-SELL layout (tsell.h): one lane per row, slot(i, w) = ((i>>5) W + w) 32 + (i&31)
struct TDev {
  int W, c0, WA, words;
  const int32_t *off;     // W template offsets
  const int32_t *offA;    // WA offsets of A's sub-template
  const int8_t *w2a;      // W -> A index or -1
  const unsigned long long *mask;  // presence bits, [slice][word][lane]
  const int32_t *asrc;    // [slice][a][lane]: index of A's entry in the local A arrays, or -1
};

// A's CSR values -> template slots aT (nslices * WA * 32), rows [0, nrows)
cudaError_t launch_tsell_gather_a(const TDev &t, const double *aval, int64_t nrows, double *aT,
                                  cudaStream_t st);
// same for local rows [r0, r1) only
// multi-GPU factor halo (template layout): columns [c0, W) of nslices slices from slice0 into a
// contiguous buffer, and back into the ghost slices (+ the compact diagonal copy udiag)
cudaError_t launch_tsell_pack_upper(const double *vals, int64_t slice0, int64_t nslices, int W,
                                    int c0, double *buf, cudaStream_t st);
cudaError_t launch_tsell_unpack_upper(const double *buf, int64_t slice0, int64_t nslices, int W,
                                      int c0, double *vals, double *udiag, cudaStream_t st);
cudaError_t launch_tsell_gather_a_range(const TDev &t, const double *aval, int64_t r0,
                                        int64_t r1, double *aT, cudaStream_t st);
cudaError_t launch_tsell_init(const TDev &t, const double *aT, const double *s,
                              const double *ad, int64_t r0, int64_t r1, double *ahatT,
                              double *vals, double *udiag, ErrFlags *err, double shift,
                              cudaStream_t st, bool iter0 = true);
cudaError_t launch_tsell_jacobi(const TDev &t, bool lower, const double *vals,
                                const double *udiag, const double *rhs, const double *xo,
                                double *xn, double *xfinal, const double *s, int64_t r0,
                                int64_t r1, int64_t Gh, double omega, bool final,
                                cudaStream_t st);
// deterministic sum of partials into *dst; also resets the tile counter (if non-null) to 0
cudaError_t launch_reduce_reset(const double *partials, int np, double *dst,
                                unsigned int *counter, cudaStream_t st);

// *dst = sum of x[i]^2 (deterministic; partials needs kSumsqBlocks entries)
constexpr int kSumsqBlocks = 256;
cudaError_t launch_sumsq(const double *x, int64_t n, double *partials, double *dst,
                         cudaStream_t st);

// ---- restarted GMRES building blocks (config 5)
constexpr int kDotBlocks = 888;  // 6 x 148: GMRES orthogonalisation grid (max)
// y[r - Gh] = sum_q aval[q] x[aci[q]] over owned rows [r0, r1) (x extended, local columns)
cudaError_t launch_spmv(const int64_t *arp, const int32_t *aci, const double *aval,
                        const double *x, double *y, int64_t r0, int64_t r1, int64_t Gh, int G,
                        cudaStream_t st);
// out[j] = V_j . w for j < k (V_j = V + j ldv), and out[k] = extra . w when extra is given (same
// pass); partials: (k + 1) * kDotBlocks doubles; out on device
cudaError_t launch_mdot(const double *V, int64_t ldv, int k, const double *w, int64_t n,
                        double *partials, double *out, cudaStream_t st,
                        const double *extra = nullptr);
// w += sign * sum_j c[j] V_j  (c on device)
cudaError_t launch_maxpy(const double *V, int64_t ldv, int k, const double *c, double *w,
                         int64_t n, double sign, cudaStream_t st);
// DCGS2 (delayed reorthogonalisation) passes, u = V_p pending: out[2 j] = V_j . u and
// out[2 j + 1] = V_j . w for j <= p (w may be null: those entries are 0); partials: 2 (p + 1)
// * kDotBlocks doubles; out on device
cudaError_t launch_dcgs_dot(const double *V, int64_t ldv, int p, const double *w, int64_t n,
                            double *partials, double *out, cudaStream_t st);
// coef (device) = [s_0..s_{p-1}, z_0..z_{p-1}, c_p, 1/rho]: V_p = (V_p - sum s_j V_j) / rho,
// V_{p+1} = (w - sum z_j V_j - c_p V_p) / rho, in one pass over V_0..V_{p-1}
cudaError_t launch_dcgs_update(double *V, int64_t ldv, int p, const double *coef, const double *w,
                               int64_t n, cudaStream_t st);
// y = a x + b y
cudaError_t launch_axpby(double a, const double *x, double b, double *y, int64_t n,
                         cudaStream_t st);

// ---- block path (bsr.cu): S made of dense BS x BS blocks (BS = 2, 3, 4), single GPU.
// Blocks stored contiguously, ST = BS*BS rounded up to even doubles per block; block b of block
// row I covers scalar rows BS I .. BS I + BS - 1 and columns BS bcol[b] ...
struct BsrDev {
  int bs;
  int64_t nb, nblk;
  const int64_t *bptr;   // nb + 1
  const int32_t *brow;   // nblk: block row of each block
  const int32_t *bcol;   // nblk
  const int32_t *bdiag;  // nb: index of the diagonal block of each block row
  const int64_t *tptr;   // nblk + 1: term range of each target block
  const int2 *terms;     // (block (I,K), block (K,J)), K ascending, K < min(I, J)
};
// smem > 0: stage each tile's block rows in smem bytes of shared memory (when they fit)
// minb: __launch_bounds__ resident-CTA hint (1 or 4)
cudaError_t bsr_sweep_occupancy(int bs, int threads, size_t smem, int minb, int *blocks_per_sm);
// asynchronous in-place block sweep: nb consecutive target blocks per thread;
// grid blocks of 256 threads, partials[grid]
cudaError_t launch_bsr_sweep_async(const BsrDev &B, const double *ahb, double *vals, double omega,
                                   double *partials, ErrFlags *err, int grid, int nb,
                                   cudaStream_t st);
cudaError_t launch_bsr_sweep(const BsrDev &B, const double *ahb, const double *old, double *out,
                             double omega, double *partials, ErrFlags *err, int grid,
                             int threads, size_t smem, int minb, cudaStream_t st);
int bsr_block_stride(int bs);
cudaError_t launch_bsr_from_csr(const BsrDev &B, const int64_t *rp, const double *vals,
                                double *vb, int64_t nrows, cudaStream_t st);
cudaError_t launch_bsr_to_csr(const BsrDev &B, const int64_t *rp, const double *vb, double *vals,
                              double *ud, int64_t nrows, cudaStream_t st);
cudaError_t launch_bsr_ahat(const BsrDev &B, const int64_t *arp, const int32_t *apos,
                            const double *ahatA, double *ahb, int64_t nrows, cudaStream_t st);

int sm_count(int device);
// raise a kernel's dynamic shared memory limit to the device's opt-in maximum
cudaError_t allow_dynamic_smem(const void *func);

}  // namespace fastilu
