// CUDA kernels of libfastilu_b200 (sm_100a).  All arithmetic fp64.
//
// Step map (PAPER.md citations at each kernel):
//   a2 scale_kernel      s_i = 1/sqrt(|a_ii|), ahat_ii                     (R5)
//   a3 init_kernel       ahat on S, L0 = ahat_ij/ahat_jj, U0 = ahat_ij     (R4)
//   a4/a5 sweep_kernel   one synchronous FastILU sweep + residual partials
//   a8 jacobi_L_kernel   z <- y - (L - I) z
//   a9 jacobi_U_kernel   w <- D^-1 (z - (U - D) w), last sweep x = s o w
//
// Factor arithmetic uses explicitly rounded __dmul_rn / __dsub_rn / __ddiv_rn in the oracle's
// order (pivots k ascending for every target), so no multiply-subtract is contracted.
#include <cooperative_groups.h>
#include <cooperative_groups/reduce.h>
#include <cooperative_groups/scan.h>

#include "device.h"

namespace cg = cooperative_groups;

namespace fastilu {

int sm_count(int device) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  return v;
}

static __device__ __forceinline__ bool bad_pivot(double d) { return !(d != 0.0 && isfinite(d)); }

// ----------------------------------------------------------------------------------------
// a2: diagonal scaling, one thread per local row.
// ----------------------------------------------------------------------------------------
__global__ void scale_kernel(const int64_t *__restrict__ arp, const int32_t *__restrict__ adiag,
                             const double *__restrict__ aval, int64_t r0, int64_t r1,
                             double *__restrict__ s, double *__restrict__ ad, ErrFlags *err) {
  for (int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < r1;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double a = aval[arp[r] + adiag[r]];
    if (a == 0.0) atomicMin(&err->zero_diag, (unsigned long long)r);
    const double si = __ddiv_rn(1.0, __dsqrt_rn(fabs(a)));
    s[r] = si;
    ad[r] = __dmul_rn(__dmul_rn(a, si), si);
  }
}

cudaError_t launch_scale(const int64_t *arp, const int32_t *adiag, const double *aval,
                         int64_t r0, int64_t r1, double *s, double *ad, ErrFlags *err,
                         cudaStream_t st) {
  if (r1 <= r0) return cudaSuccess;
  int64_t blocks = (r1 - r0 + 255) / 256;
  if (blocks > 65535 * 16) blocks = 65535 * 16;
  scale_kernel<<<(unsigned)blocks, 256, 0, st>>>(arp, adiag, aval, r0, r1, s, ad, err);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------------------
// a3: scaled values on S and the initial guess; one G-lane group per owned row.
// ----------------------------------------------------------------------------------------
template <int G>
__global__ void __launch_bounds__(256)
init_kernel(DevPattern P, const int64_t *__restrict__ arp, const int32_t *__restrict__ aci,
            const int32_t *__restrict__ apos, const double *__restrict__ aval,
            const double *__restrict__ s, const double *__restrict__ ad, int64_t r0, int64_t r1,
            double *__restrict__ ahat, double *__restrict__ vals, double *__restrict__ udiag,
            ErrFlags *err) {
  auto tile = cg::tiled_partition<G>(cg::this_thread_block());
  const int gpb = blockDim.x / G;
  const int lane = tile.thread_rank();
  const int64_t stride = (int64_t)gridDim.x * gpb;
  for (int64_t row = r0 + (int64_t)blockIdx.x * gpb + threadIdx.x / G; row < r1; row += stride) {
    const int64_t rb = P.rp[row], re = P.rp[row + 1];
    for (int64_t p = rb + lane; p < re; p += G) {
      ahat[p] = 0.0;  // fill entries: +0.0 (R4)
      vals[p] = 0.0;
    }
    tile.sync();
    const double si = s[row];
    for (int64_t q = arp[row] + lane; q < arp[row + 1]; q += G) {
      const int32_t j = aci[q];
      const int64_t p = rb + apos[q];
      const double ah = __dmul_rn(__dmul_rn(aval[q], si), s[j]);
      ahat[p] = ah;
      vals[p] = (j < row) ? __ddiv_rn(ah, ad[j]) : ah;
      if (j == row) {
        udiag[row] = ah;
        if (bad_pivot(ah)) atomicMin(&err->zero_pivot, (unsigned long long)row);
      }
    }
    tile.sync();
  }
}

cudaError_t launch_init(const DevPattern &P, const int64_t *arp, const int32_t *aci,
                        const int32_t *apos, const double *aval, const double *s,
                        const double *ad, int64_t r0, int64_t r1, double *ahat, double *vals,
                        double *udiag, ErrFlags *err, int G, cudaStream_t st) {
  if (r1 <= r0) return cudaSuccess;
  const int threads = 256, gpb = threads / G;
  int64_t blocks = (r1 - r0 + gpb - 1) / gpb;
  if (blocks > (1ll << 30)) blocks = 1ll << 30;
#define FASTILU_INIT(GG)                                                                   \
  init_kernel<GG><<<(unsigned)blocks, threads, 0, st>>>(P, arp, aci, apos, aval, s, ad, r0, r1, \
                                                         ahat, vals, udiag, err)
  switch (G) {
    case 4: FASTILU_INIT(4); break;
    case 8: FASTILU_INIT(8); break;
    case 16: FASTILU_INIT(16); break;
    default: FASTILU_INIT(32); break;
  }
#undef FASTILU_INIT
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------------------
// a4 + a5: one synchronous FastILU sweep (readings R1-R3), row-oriented.
//
// For row i the group computes every entry of S_i at once:
//   acc[p] = ahat_ip;  for each pivot k in L_i ascending (k = S_i[t], t < nl):
//       for each j in the strict upper row of U_k (j > k) with (i,j) in S:
//           acc[p(j)] -= l_ik * u_kj                      (old values, iterate s-1)
// which is exactly the oracle's sum over k < min(i,j), (k,j) in S, in ascending k, for every
// target.  The U-rows of a chunk of P pivots are staged in shared memory by one flattened,
// coalesced copy (all loads in flight at once), then applied pivot by pivot.
// Finalize: l_ij = acc / u_jj(old), u_ij = acc (omega-damped), residual partial
// (acc - l_ij u_jj)^2 / (acc - u_ij)^2 of iterate s-1, new diagonal copied to udiag.
// ----------------------------------------------------------------------------------------
__host__ __device__ inline size_t sweep_group_bytes(int cap_m, int cap_st, int Pv) {
  size_t b = (size_t)cap_m * 12 + (size_t)cap_st * 12 + (size_t)Pv * 16 + (size_t)(Pv + 1) * 4;
  return (b + 15) & ~(size_t)15;
}

template <int G>
__global__ void __launch_bounds__(256)
sweep_kernel(DevPattern P, const double *__restrict__ ahat, const double *__restrict__ old,
             double *__restrict__ out, const double *__restrict__ udo, double *__restrict__ udn,
             int64_t r0, int64_t r1, double omega, double *__restrict__ partials, ErrFlags *err,
             int cap_m, int Pv, int cap_st) {
  extern __shared__ __align__(16) unsigned char smem[];
  auto blk = cg::this_thread_block();
  auto tile = cg::tiled_partition<G>(blk);
  const int gpb = blockDim.x / G;
  const int gib = threadIdx.x / G;
  const int lane = tile.thread_rank();
  unsigned char *gb = smem + sweep_group_bytes(cap_m, cap_st, Pv) * gib;
  double *acc = reinterpret_cast<double *>(gb);
  double *stv = acc + cap_m;
  double *lik = stv + cap_st;
  int64_t *ub = reinterpret_cast<int64_t *>(lik + Pv);
  int32_t *sc = reinterpret_cast<int32_t *>(ub + Pv);
  int32_t *stc = sc + cap_m;
  int32_t *off = stc + cap_st;
  const bool damp = (omega != 1.0);
  const double om1 = 1.0 - omega;

  double r2 = 0.0;
  const int64_t stride = (int64_t)gridDim.x * gpb;
  for (int64_t row = r0 + (int64_t)blockIdx.x * gpb + gib; row < r1; row += stride) {
    const int64_t rb = P.rp[row];
    const int m = (int)(P.rp[row + 1] - rb);
    const int nl = P.dloc[row];
    for (int p = lane; p < m; p += G) {
      sc[p] = P.ci[rb + p];
      acc[p] = ahat[rb + p];
    }
    tile.sync();
    for (int t0 = 0; t0 < nl; t0 += Pv) {
      const int np = min(Pv, nl - t0);
      int len = 0;
      if (lane < np) {
        const int k = sc[t0 + lane];
        const int64_t u0 = P.rp[k] + P.dloc[k] + 1;  // strict upper part of row k
        len = (int)(P.rp[k + 1] - u0);
        ub[lane] = u0;
        lik[lane] = old[rb + t0 + lane];
      }
      const int incl = cg::inclusive_scan(tile, len);
      if (lane < np) off[lane] = incl - len;
      const int total = tile.shfl(incl, np - 1);
      if (lane == 0) off[np] = total;
      tile.sync();
      for (int c = lane; c < total; c += G) {
        int lo = 0, hi = np;  // off[lo] <= c < off[lo + 1]
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (off[mid] <= c) lo = mid; else hi = mid;
        }
        const int64_t src = ub[lo] + (c - off[lo]);
        stc[c] = P.ci[src];
        stv[c] = old[src];
      }
      tile.sync();
      for (int q = 0; q < np; q++) {
        const double l = lik[q];
        const int t = t0 + q;
        const int e1 = off[q + 1];
        for (int e = off[q] + lane; e < e1; e += G) {
          const int j = stc[e];
          int lo = t + 1, hi = m - 1, p = -1;
          while (lo <= hi) {
            const int mid = (lo + hi) >> 1;
            const int cm = sc[mid];
            if (cm == j) { p = mid; break; }
            if (cm < j) lo = mid + 1; else hi = mid - 1;
          }
          if (p >= 0) acc[p] = __dsub_rn(acc[p], __dmul_rn(l, stv[e]));
        }
        tile.sync();
      }
    }
    for (int p = lane; p < m; p += G) {
      const double a = acc[p];
      const double o = old[rb + p];
      double nv, e;
      if (p < nl) {
        const double ujj = udo[sc[p]];
        e = __dsub_rn(a, __dmul_rn(o, ujj));
        const double l = __ddiv_rn(a, ujj);
        nv = damp ? __dadd_rn(__dmul_rn(om1, o), __dmul_rn(omega, l)) : l;
      } else {
        e = __dsub_rn(a, o);
        nv = damp ? __dadd_rn(__dmul_rn(om1, o), __dmul_rn(omega, a)) : a;
      }
      r2 = fma(e, e, r2);
      out[rb + p] = nv;
      if (p == nl) {
        udn[row] = nv;
        if (bad_pivot(nv)) atomicMin(&err->zero_pivot, (unsigned long long)row);
      }
    }
    tile.sync();
  }
  // deterministic block reduction of r2 (fixed shuffle tree, then warps in order)
  __shared__ double wsum[32];
  double v = r2;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += wsum[w];
    partials[blockIdx.x] = t;
  }
}

template <int G>
static cudaError_t launch_sweep_t(const DevPattern &P, const double *ahat, const double *old,
                                  double *out, const double *udo, double *udn, int64_t r0,
                                  int64_t r1, double omega, double *partials, ErrFlags *err,
                                  const SweepCfg &c, cudaStream_t st) {
  static bool attr_set = false;
  static size_t attr_bytes = 0;
  if (!attr_set || attr_bytes < c.smem) {
    cudaFuncSetAttribute(sweep_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(c.smem > 48 * 1024 ? c.smem : 48 * 1024));
    attr_set = true;
    attr_bytes = c.smem;
  }
  sweep_kernel<G><<<c.grid, c.warps * 32, c.smem, st>>>(P, ahat, old, out, udo, udn, r0, r1,
                                                         omega, partials, err, c.cap_m, c.P,
                                                         c.cap_st);
  return cudaGetLastError();
}

cudaError_t launch_sweep(const DevPattern &P, const double *ahat, const double *old,
                         double *out, const double *udiag_old, double *udiag_new, int64_t r0,
                         int64_t r1, double omega, double *partials, ErrFlags *err,
                         const SweepCfg &cfg, cudaStream_t st) {
  switch (cfg.G) {
    case 4: return launch_sweep_t<4>(P, ahat, old, out, udiag_old, udiag_new, r0, r1, omega,
                                      partials, err, cfg, st);
    case 8: return launch_sweep_t<8>(P, ahat, old, out, udiag_old, udiag_new, r0, r1, omega,
                                      partials, err, cfg, st);
    case 16: return launch_sweep_t<16>(P, ahat, old, out, udiag_old, udiag_new, r0, r1, omega,
                                        partials, err, cfg, st);
    default: return launch_sweep_t<32>(P, ahat, old, out, udiag_old, udiag_new, r0, r1, omega,
                                        partials, err, cfg, st);
  }
}

// deterministic sum of the per-block partials (one block, fixed order)
__global__ void reduce_kernel(const double *__restrict__ partials, int np, double *dst) {
  __shared__ double sh[1024];
  double t = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) t += partials[i];
  sh[threadIdx.x] = t;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *dst = sh[0];
}

cudaError_t launch_reduce(const double *partials, int np, double *dst, cudaStream_t st) {
  reduce_kernel<<<1, 1024, 0, st>>>(partials, np, dst);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------------------
// a8 / a9: FastSpTRSV Jacobi sweeps (out of place per PAPER.md:717; R6).
// ----------------------------------------------------------------------------------------
__global__ void first_L_kernel(const double *__restrict__ b, const double *__restrict__ s,
                               double *__restrict__ y, double *__restrict__ z, int64_t r0,
                               int64_t r1, int64_t G, double omega) {
  for (int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < r1;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double yi = __dmul_rn(s[r], b[r - G]);
    y[r] = yi;
    z[r] = (omega == 1.0) ? yi : __dmul_rn(omega, yi);  // z1 = (1-w) 0 + w y
  }
}

__global__ void first_U_kernel(const double *__restrict__ z, const double *__restrict__ ud,
                               const double *__restrict__ s, double *__restrict__ w,
                               double *__restrict__ x, int64_t r0, int64_t r1, int64_t G,
                               double omega, bool final) {
  for (int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < r1;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double u = __ddiv_rn(z[r], ud[r]);
    const double wi = (omega == 1.0) ? u : __dmul_rn(omega, u);
    if (final) x[r - G] = __dmul_rn(s[r], wi); else w[r] = wi;
  }
}

static unsigned vec_blocks(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 65535 * 16) b = 65535 * 16;
  return (unsigned)(b > 0 ? b : 1);
}

cudaError_t launch_trisolve_first_L(const double *b, const double *s, double *y, double *z,
                                    int64_t r0, int64_t r1, int64_t G, double omega,
                                    cudaStream_t st) {
  if (r1 <= r0) return cudaSuccess;
  first_L_kernel<<<vec_blocks(r1 - r0), 256, 0, st>>>(b, s, y, z, r0, r1, G, omega);
  return cudaGetLastError();
}

cudaError_t launch_trisolve_first_U(const double *z, const double *udiag, const double *s,
                                    double *w, double *x, int64_t r0, int64_t r1, int64_t G,
                                    double omega, bool final, cudaStream_t st) {
  if (r1 <= r0) return cudaSuccess;
  first_U_kernel<<<vec_blocks(r1 - r0), 256, 0, st>>>(z, udiag, s, w, x, r0, r1, G, omega,
                                                       final);
  return cudaGetLastError();
}

template <int G, bool LOWER>
__global__ void __launch_bounds__(256)
jacobi_kernel(DevPattern P, const double *__restrict__ vals, const double *__restrict__ ud,
              const double *__restrict__ rhs, const double *__restrict__ xo,
              double *__restrict__ xn, double *__restrict__ xfinal, const double *__restrict__ s,
              int64_t r0, int64_t r1, int64_t Gh, double omega, bool final) {
  auto tile = cg::tiled_partition<G>(cg::this_thread_block());
  const int gpb = blockDim.x / G;
  const int lane = tile.thread_rank();
  const int64_t stride = (int64_t)gridDim.x * gpb;
  for (int64_t row = r0 + (int64_t)blockIdx.x * gpb + threadIdx.x / G; row < r1; row += stride) {
    const int64_t rb = P.rp[row];
    const int nl = P.dloc[row];
    const int64_t b0 = LOWER ? rb : rb + nl + 1;
    const int64_t b1 = LOWER ? rb + nl : P.rp[row + 1];
    double sum = 0.0;
    for (int64_t p = b0 + lane; p < b1; p += G) sum = fma(vals[p], xo[P.ci[p]], sum);
    sum = cg::reduce(tile, sum, cg::plus<double>());
    if (lane == 0) {
      double u = rhs[row] - sum;
      if (!LOWER) u = __ddiv_rn(u, ud[row]);
      const double v = (omega == 1.0) ? u : (1.0 - omega) * xo[row] + omega * u;
      if (final) xfinal[row - Gh] = __dmul_rn(s[row], v); else xn[row] = v;
    }
  }
}

template <bool LOWER>
static cudaError_t launch_jacobi_t(const DevPattern &P, const double *vals, const double *ud,
                                   const double *rhs, const double *xo, double *xn, double *xf,
                                   const double *s, int64_t r0, int64_t r1, int64_t Gh,
                                   double omega, bool final, int G, cudaStream_t st) {
  if (r1 <= r0) return cudaSuccess;
  const int threads = 256, gpb = threads / G;
  int64_t blocks = (r1 - r0 + gpb - 1) / gpb;
  if (blocks > (1ll << 30)) blocks = 1ll << 30;
#define FASTILU_JAC(GG)                                                                     \
  jacobi_kernel<GG, LOWER><<<(unsigned)blocks, threads, 0, st>>>(P, vals, ud, rhs, xo, xn, xf, s, \
                                                                   r0, r1, Gh, omega, final)
  switch (G) {
    case 1: FASTILU_JAC(1); break;
    case 2: FASTILU_JAC(2); break;
    case 4: FASTILU_JAC(4); break;
    case 8: FASTILU_JAC(8); break;
    case 16: FASTILU_JAC(16); break;
    default: FASTILU_JAC(32); break;
  }
#undef FASTILU_JAC
  return cudaGetLastError();
}

cudaError_t launch_jacobi_L(const DevPattern &P, const double *vals, const double *y,
                            const double *zold, double *znew, int64_t r0, int64_t r1,
                            double omega, int G, cudaStream_t st) {
  return launch_jacobi_t<true>(P, vals, nullptr, y, zold, znew, nullptr, nullptr, r0, r1, 0,
                               omega, false, G, st);
}

cudaError_t launch_jacobi_U(const DevPattern &P, const double *vals, const double *udiag,
                            const double *z, const double *wold, double *wnew, double *x,
                            const double *s, int64_t r0, int64_t r1, int64_t Gh, double omega,
                            bool final, int G, cudaStream_t st) {
  return launch_jacobi_t<false>(P, vals, udiag, z, wold, wnew, x, s, r0, r1, Gh, omega, final,
                                G, st);
}

}  // namespace fastilu
