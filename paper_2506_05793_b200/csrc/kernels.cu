// CUDA kernels of libfastilu_b200 (sm_100a).  All arithmetic fp64.
//
// Step map (PAPER.md citations at each kernel):
//   a2 scale_kernel      s_i = 1/sqrt(|a_ii|), ahat_ii                     (R5)
//   a3 init_kernel       ahat on A, L0 = ahat_ij/ahat_jj, U0 = ahat_ij     (R4)
//   a4/a5 sweep_kernel   one synchronous FastILU sweep + residual partials
//   a8 jacobi_L_kernel   z <- y - (L - I) z
//   a9 jacobi_U_kernel   w <- D^-1 (z - (U - D) w), last sweep x = s o w
//
// Factor arithmetic uses explicitly rounded __dmul_rn / __dsub_rn / __ddiv_rn in the oracle's
// order (pivots k ascending for every target), so no multiply-subtract is contracted.
#include <cooperative_groups.h>
#include <cooperative_groups/reduce.h>
#include <cooperative_groups/scan.h>

#include <algorithm>

#include "device.h"

namespace cg = cooperative_groups;

namespace fastilu {

// The dynamic-smem limit is a property of the kernel function, shared by every handle: raise it
// to the device's opt-in maximum (monotone) instead of the calling handle's need, so a handle
// configured later with less shared memory cannot break the launches of an earlier one.
cudaError_t allow_dynamic_smem(const void *func) {
  int dev = 0, mx = 0;
  cudaGetDevice(&dev);
  cudaError_t e = cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa{};
  e = cudaFuncGetAttributes(&fa, func);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              mx - (int)fa.sharedSizeBytes);  // static + dynamic <= opt-in max
}

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
                             double *__restrict__ s, double *__restrict__ ad, ErrFlags *err,
                             double shift) {
  for (int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < r1;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double a0 = aval[arp[r] + adiag[r]];
    const double a = __dadd_rn(a0, __dmul_rn(shift, fabs(a0)));  // Manteuffel: a + alpha |a|
    if (a == 0.0) atomicMin(&err->zero_diag, (unsigned long long)r);
    const double si = __ddiv_rn(1.0, __dsqrt_rn(fabs(a)));
    s[r] = si;
    ad[r] = __dmul_rn(__dmul_rn(a, si), si);
  }
}

cudaError_t launch_scale(const int64_t *arp, const int32_t *adiag, const double *aval,
                         int64_t r0, int64_t r1, double *s, double *ad, ErrFlags *err,
                         double shift, cudaStream_t st) {
  if (r1 <= r0) return cudaSuccess;
  int64_t blocks = (r1 - r0 + 255) / 256;
  if (blocks > 65535 * 16) blocks = 65535 * 16;
  scale_kernel<<<(unsigned)blocks, 256, 0, st>>>(arp, adiag, aval, r0, r1, s, ad, err, shift);
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
            double *__restrict__ ahatA, double *__restrict__ vals, double *__restrict__ udiag,
            ErrFlags *err, double shift) {
  auto tile = cg::tiled_partition<G>(cg::this_thread_block());
  const int gpb = blockDim.x / G;
  const int lane = tile.thread_rank();
  const int64_t stride = (int64_t)gridDim.x * gpb;
  for (int64_t row = r0 + (int64_t)blockIdx.x * gpb + threadIdx.x / G; row < r1; row += stride) {
    const int64_t rb = P.rp[row], re = P.rp[row + 1];
    for (int64_t p = rb + lane; p < re; p += G) vals[p] = 0.0;  // fill entries: +0.0 (R4)
    tile.sync();
    const double si = s[row];
    for (int64_t q = arp[row] + lane; q < arp[row + 1]; q += G) {
      const int32_t j = aci[q];
      const int64_t p = rb + apos[q];
      const double av = (j == row) ? __dadd_rn(aval[q], __dmul_rn(shift, fabs(aval[q]))) : aval[q];
      const double ah = __dmul_rn(__dmul_rn(av, si), s[j]);
      ahatA[q] = ah;
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
                        const double *ad, int64_t r0, int64_t r1, double *ahatA, double *vals,
                        double *udiag, ErrFlags *err, int G, double shift, cudaStream_t st) {
  if (r1 <= r0) return cudaSuccess;
  const int threads = 256, gpb = threads / G;
  int64_t blocks = (r1 - r0 + gpb - 1) / gpb;
  if (blocks > (1ll << 30)) blocks = 1ll << 30;
#define FASTILU_INIT(GG)                                                                   \
  init_kernel<GG><<<(unsigned)blocks, threads, 0, st>>>(P, arp, aci, apos, aval, s, ad, r0, r1, \
                                                         ahatA, vals, udiag, err, shift)
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
// target (the same rounded products subtracted in the same order => bitwise equal).
//  * the row's columns, its accumulator (seeded from ahat on A's pattern) and a position table
//    live in shared memory; p(j) is found through an injective multiplicative hash of the
//    offset j - i (verified on the host for every row at create) or, if none was found, by
//    binary search;
//  * lanes take consecutive entries of U_k (coalesced); the next pivot's entries are loaded
//    into registers while the current pivot is applied (software pipeline, no smem staging);
//  * each block owns a contiguous chunk of rows and its groups walk it interleaved, so
//    neighbouring rows (which share most of their pivots' U-rows) run on the same SM (L1).
// Finalize: l_ij = acc / u_jj(old), u_ij = acc (omega-damped), residual partial of iterate s-1
// ((acc - l_ij u_jj)^2 or (acc - u_ij)^2), contiguous row write, diagonal copy into udiag.
// ----------------------------------------------------------------------------------------
__host__ __device__ inline size_t sweep_group_bytes(int cap_m, int hsize) {
  size_t b = (size_t)cap_m * 12 + (size_t)hsize * 2;
  return (b + 15) & ~(size_t)15;
}

template <int G, bool HASH>
__global__ void __launch_bounds__(512)
sweep_kernel(DevPattern P, const int64_t *__restrict__ arp, const int32_t *__restrict__ apos,
             const double *__restrict__ ahatA, const double *__restrict__ old,
             double *__restrict__ out, const double *__restrict__ udo, double *__restrict__ udn,
             int64_t r0, int64_t r1, int64_t chunk, double omega, double *__restrict__ partials,
             ErrFlags *err, int cap_m, uint32_t hmul, int hshift, int hsize) {
  extern __shared__ __align__(16) unsigned char smem[];
  auto blk = cg::this_thread_block();
  auto tile = cg::tiled_partition<G>(blk);
  const int gpb = blockDim.x / G;
  const int gib = threadIdx.x / G;
  const int lane = tile.thread_rank();
  unsigned char *gb = smem + sweep_group_bytes(cap_m, hsize) * gib;
  double *acc = reinterpret_cast<double *>(gb);
  int32_t *sc = reinterpret_cast<int32_t *>(acc + cap_m);
  uint16_t *T = reinterpret_cast<uint16_t *>(sc + cap_m);
  const bool damp = (omega != 1.0);
  const double om1 = 1.0 - omega;

  double r2 = 0.0;
  // tile-strided rows: block b takes tiles of `chunk` consecutive rows, tiles strided by the
  // grid, so all SMs work inside one window of grid*chunk rows (the pivots' U-rows stay in
  // L2) while each block walks consecutive rows (neighbours share U-rows in L1).
  for (int64_t row = r0 + (int64_t)blockIdx.x * chunk + gib; row < r1;
       row += ((row - r0) % chunk + gpb < chunk) ? gpb
                                                 : (int64_t)(gridDim.x - 1) * chunk + gpb) {
    const int64_t rb = P.rp[row];
    const int m = (int)(P.rp[row + 1] - rb);
    const int nl = P.dloc[row];
    const int irow = (int)row;
    for (int p = lane; p < m; p += G) {
      const int c = P.ci[rb + p];
      sc[p] = c;
      acc[p] = 0.0;  // fill entries start from +0.0 (R4)
      if (HASH) T[((uint32_t)(c - irow) * hmul) >> hshift] = (uint16_t)p;
    }
    tile.sync();
    for (int64_t q = arp[row] + lane; q < arp[row + 1]; q += G) acc[apos[q]] = ahatA[q];
    tile.sync();

    auto apply1 = [&](int j, double u, double l, int t) {
      int p = -1;
      if (HASH) {
        const int pp = T[((uint32_t)(j - irow) * hmul) >> hshift];
        if (pp < m && sc[pp] == j) p = pp;
      } else {
        int lo = t + 1, hi = m - 1;
        while (lo <= hi) {
          const int mid = (lo + hi) >> 1;
          const int cm = sc[mid];
          if (cm == j) { p = mid; break; }
          if (cm < j) lo = mid + 1; else hi = mid - 1;
        }
      }
      if (p >= 0) acc[p] = __dsub_rn(acc[p], __dmul_rn(l, u));
    };

    for (int t0 = 0; t0 < nl; t0 += G) {
      const int np = min(G, nl - t0);
      int64_t ub = 0;
      int len = 0;
      double lv = 0.0;
      if (lane < np) {
        const int k = sc[t0 + lane];
        const int64_t rk = P.rp[k];
        ub = rk + P.dloc[k] + 1;  // strict upper part of row k
        len = (int)(P.rp[k + 1] - ub);
        lv = old[rb + t0 + lane];
      }
      // software pipeline: (cj0,cu0),(cj1,cu1) = entries lane, lane+G of the current pivot
      int64_t cbse = tile.shfl(ub, 0);
      int clen = tile.shfl(len, 0);
      double cl = tile.shfl(lv, 0);
      int cj0 = -1, cj1 = -1;
      double cu0 = 0.0, cu1 = 0.0;
      if (lane < clen) { cj0 = P.ci[cbse + lane]; cu0 = old[cbse + lane]; }
      if (lane + G < clen) { cj1 = P.ci[cbse + lane + G]; cu1 = old[cbse + lane + G]; }
      for (int q = 0; q < np; q++) {
        int64_t nbse = 0;
        int nlen = 0;
        double nlv = 0.0;
        int nj0 = -1, nj1 = -1;
        double nu0 = 0.0, nu1 = 0.0;
        if (q + 1 < np) {
          nbse = tile.shfl(ub, q + 1);
          nlen = tile.shfl(len, q + 1);
          nlv = tile.shfl(lv, q + 1);
          if (lane < nlen) { nj0 = P.ci[nbse + lane]; nu0 = old[nbse + lane]; }
          if (lane + G < nlen) { nj1 = P.ci[nbse + lane + G]; nu1 = old[nbse + lane + G]; }
        }
        const int t = t0 + q;
        if (cj0 >= 0) apply1(cj0, cu0, cl, t);
        if (cj1 >= 0) apply1(cj1, cu1, cl, t);
        for (int e = lane + 2 * G; e < clen; e += G) apply1(P.ci[cbse + e], old[cbse + e], cl, t);
        tile.sync();
        cbse = nbse; clen = nlen; cl = nlv;
        cj0 = nj0; cj1 = nj1; cu0 = nu0; cu1 = nu1;
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

template <int G, bool HASH>
static cudaError_t launch_sweep_t(const SweepArgs &a, const SweepCfg &c, cudaStream_t st) {
  sweep_kernel<G, HASH><<<c.grid, c.threads, c.smem, st>>>(
      a.P, a.arp, a.apos, a.ahatA, a.old, a.out, a.udo, a.udn, a.r0, a.r1, c.chunk, a.omega,
      a.partials, a.err, c.cap_m, c.hmul, c.hshift, c.hsize);
  return cudaGetLastError();
}

template <int G, bool HASH>
static cudaError_t sweep_attr_t(const SweepCfg &c, int *blocks_per_sm) {
  cudaError_t e = allow_dynamic_smem((const void *)sweep_kernel<G, HASH>);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, sweep_kernel<G, HASH>,
                                                       c.threads, c.smem);
}

#define FASTILU_SWEEP_DISPATCH(FN, ...)                                   \
  switch (cfg.G) {                                                        \
    case 4: return cfg.hash ? FN<4, true>(__VA_ARGS__) : FN<4, false>(__VA_ARGS__);     \
    case 8: return cfg.hash ? FN<8, true>(__VA_ARGS__) : FN<8, false>(__VA_ARGS__);     \
    case 16: return cfg.hash ? FN<16, true>(__VA_ARGS__) : FN<16, false>(__VA_ARGS__);  \
    default: return cfg.hash ? FN<32, true>(__VA_ARGS__) : FN<32, false>(__VA_ARGS__);  \
  }

cudaError_t sweep_configure(const SweepCfg &cfg, int *blocks_per_sm) {
  FASTILU_SWEEP_DISPATCH(sweep_attr_t, cfg, blocks_per_sm)
}

cudaError_t launch_sweep(const SweepArgs &a, const SweepCfg &cfg, cudaStream_t st) {
  FASTILU_SWEEP_DISPATCH(launch_sweep_t, a, cfg, st)
}

// ----------------------------------------------------------------------------------------
// a4 + a5, class-program variant (classes.cpp): the same recurrence in the same order, with
// the index matching precomputed per structure class.  Per pivot t of row i, lane e loads
// u_k,e (coalesced, L1/L2) and the byte prog[class][t][e] = position of (i, j_e) in S_i
// (255 = not in S), then acc[p] -= l_ik u_kj.  No column loads, hashing or searching.
// ----------------------------------------------------------------------------------------
__host__ __device__ inline size_t prog_group_bytes(int cap_m, int G) {
  size_t b = (size_t)cap_m * 8 + (size_t)G * 24;
  return (b + 15) & ~(size_t)15;
}

template <int G, int E>
__global__ void __launch_bounds__(512)
sweep_prog_kernel(DevPattern P, ProgView pv, const int64_t *__restrict__ arp,
                  const double *__restrict__ ahatA, const double *__restrict__ old,
                  double *__restrict__ out, const double *__restrict__ udo,
                  double *__restrict__ udn, int64_t r0, int64_t r1, int64_t chunk, double omega,
                  double *__restrict__ partials, ErrFlags *err, int cap_m) {
  extern __shared__ __align__(16) unsigned char smem[];
  auto blk = cg::this_thread_block();
  auto tile = cg::tiled_partition<G>(blk);
  const int gpb = blockDim.x / G;
  const int gib = threadIdx.x / G;
  const int lane = tile.thread_rank();
  unsigned char *gb = smem + prog_group_bytes(cap_m, G) * gib;
  double *acc = reinterpret_cast<double *>(gb);
  int64_t *pub = reinterpret_cast<int64_t *>(acc + cap_m);  // pivot U-row starts
  double *plv = reinterpret_cast<double *>(pub + G);        // l_ik
  int32_t *plen = reinterpret_cast<int32_t *>(plv + G);     // U-row lengths
  int32_t *poff = plen + G;                                 // program offsets
  const bool damp = (omega != 1.0);
  const double om1 = 1.0 - omega;
  const uint8_t *__restrict__ prog = pv.prog;

  double r2 = 0.0;
  // tile-strided rows: block b takes tiles of `chunk` consecutive rows, tiles strided by the
  // grid, so all SMs work inside one window of grid*chunk rows (the pivots' U-rows stay in
  // L2) while each block walks consecutive rows (neighbours share U-rows in L1).
  for (int64_t row = r0 + (int64_t)blockIdx.x * chunk + gib; row < r1;
       row += ((row - r0) % chunk + gpb < chunk) ? gpb
                                                 : (int64_t)(gridDim.x - 1) * chunk + gpb) {
    const int64_t rb = P.rp[row];
    const int m = (int)(P.rp[row + 1] - rb);
    const int nl = P.dloc[row];
    const int cls = pv.row_class[row - r0];
    const int64_t pbase = pv.class_off[cls];
    const int aoff = pv.class_aoff[cls];
    const int64_t a0 = arp[row];
    const int na = (int)(arp[row + 1] - a0);
    for (int p = lane; p < m; p += G) acc[p] = 0.0;  // fill entries start from +0.0 (R4)
    tile.sync();
    for (int q = lane; q < na; q += G) acc[prog[pbase + aoff + q]] = ahatA[a0 + q];
    int carry = 0;
    for (int t0 = 0; t0 < nl; t0 += G) {
      const int np = min(G, nl - t0);
      int len = 0;
      if (lane < np) {
        const int k = P.ci[rb + t0 + lane];
        const int64_t u0 = P.rp[k] + P.dloc[k] + 1;  // strict upper part of row k
        len = (int)(P.rp[k + 1] - u0);
        pub[lane] = u0;
        plv[lane] = old[rb + t0 + lane];
      }
      const int excl = cg::exclusive_scan(tile, len);
      if (lane < np) {
        plen[lane] = len;
        poff[lane] = carry + excl;
      }
      carry += tile.shfl(excl + len, G - 1);
      tile.sync();
      // software pipeline over the pivots: next pivot's (u, position) loaded ahead
      double cu[E];
      int cp[E];
      {
        const int64_t u0 = pub[0];
        const int L = plen[0], po = poff[0];
#pragma unroll
        for (int e = 0; e < E; e++) {
          const int idx = lane + e * G;
          cu[e] = idx < L ? old[u0 + idx] : 0.0;
          cp[e] = idx < L ? prog[pbase + po + idx] : 255;
        }
      }
      for (int q = 0; q < np; q++) {
        double nu[E];
        int npp[E];
#pragma unroll
        for (int e = 0; e < E; e++) { nu[e] = 0.0; npp[e] = 255; }
        if (q + 1 < np) {
          const int64_t u0 = pub[q + 1];
          const int L = plen[q + 1], po = poff[q + 1];
#pragma unroll
          for (int e = 0; e < E; e++) {
            const int idx = lane + e * G;
            if (idx < L) {
              nu[e] = old[u0 + idx];
              npp[e] = prog[pbase + po + idx];
            }
          }
        }
        const double l = plv[q];
#pragma unroll
        for (int e = 0; e < E; e++)
          if (cp[e] != 255) acc[cp[e]] = __dsub_rn(acc[cp[e]], __dmul_rn(l, cu[e]));
        tile.sync();
#pragma unroll
        for (int e = 0; e < E; e++) { cu[e] = nu[e]; cp[e] = npp[e]; }
      }
    }
    tile.sync();
    for (int p = lane; p < m; p += G) {
      const double a = acc[p];
      const double o = old[rb + p];
      double nv, e;
      if (p < nl) {
        const double ujj = udo[P.ci[rb + p]];
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

template <int G, int E>
static cudaError_t launch_prog_t(const SweepArgs &a, const ProgView &pv, const SweepCfg &c,
                                 cudaStream_t st) {
  sweep_prog_kernel<G, E><<<c.grid, c.threads, c.smem, st>>>(
      a.P, pv, a.arp, a.ahatA, a.old, a.out, a.udo, a.udn, a.r0, a.r1, c.chunk, a.omega,
      a.partials, a.err, c.cap_m);
  return cudaGetLastError();
}

template <int G, int E>
static cudaError_t prog_attr_t(const SweepCfg &c, int *bps) {
  cudaError_t e = allow_dynamic_smem((const void *)sweep_prog_kernel<G, E>);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, sweep_prog_kernel<G, E>, c.threads,
                                                       c.smem);
}

#define FASTILU_PROG_DISPATCH(FN, ...)                                           \
  switch (cfg.G * 8 + cfg.E) {                                                   \
    case 4 * 8 + 1: return FN<4, 1>(__VA_ARGS__);                                \
    case 4 * 8 + 2: return FN<4, 2>(__VA_ARGS__);                                \
    case 8 * 8 + 1: return FN<8, 1>(__VA_ARGS__);                                \
    case 8 * 8 + 2: return FN<8, 2>(__VA_ARGS__);                                \
    case 16 * 8 + 1: return FN<16, 1>(__VA_ARGS__);                              \
    case 16 * 8 + 2: return FN<16, 2>(__VA_ARGS__);                              \
    case 32 * 8 + 1: return FN<32, 1>(__VA_ARGS__);                              \
    case 32 * 8 + 2: return FN<32, 2>(__VA_ARGS__);                              \
    case 32 * 8 + 4: return FN<32, 4>(__VA_ARGS__);                              \
    default: return cudaErrorInvalidConfiguration;                               \
  }

cudaError_t sweep_prog_configure(const SweepCfg &cfg, int *blocks_per_sm) {
  FASTILU_PROG_DISPATCH(prog_attr_t, cfg, blocks_per_sm)
}

cudaError_t launch_sweep_prog(const SweepArgs &a, const ProgView &pv, const SweepCfg &cfg,
                              cudaStream_t st) {
  FASTILU_PROG_DISPATCH(launch_prog_t, a, pv, cfg, st)
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

// ntri = 1: the first L and the first U sweep in one pass, x = s o (w (w (s o b)) / u_ii) with
// the same rounded operations in the same order as first_L then first_U (bitwise the same x;
// y and z are not stored: nothing reads them after a one-sweep apply)
__global__ void first_LU_kernel(const double *__restrict__ b, const double *__restrict__ s,
                                const double *__restrict__ ud, double *__restrict__ x, int64_t r0,
                                int64_t r1, int64_t G, double omega) {
  for (int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < r1;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double si = s[r];
    const double yi = __dmul_rn(si, b[r - G]);
    const double zi = (omega == 1.0) ? yi : __dmul_rn(omega, yi);
    const double u = __ddiv_rn(zi, ud[r]);
    const double wi = (omega == 1.0) ? u : __dmul_rn(omega, u);
    x[r - G] = __dmul_rn(si, wi);
  }
}

cudaError_t launch_trisolve_first_LU(const double *b, const double *s, const double *udiag,
                                     double *x, int64_t r0, int64_t r1, int64_t G, double omega,
                                     cudaStream_t st) {
  if (r1 <= r0) return cudaSuccess;
  first_LU_kernel<<<vec_blocks(r1 - r0), 256, 0, st>>>(b, s, udiag, x, r0, r1, G, omega);
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

// One G-lane group per row: the lanes load G consecutive entries at a time (coalesced) and form
// the rounded products l_ij x_j; the row sum is then taken in the oracle's order (ascending
// columns, y - p_0 - p_1 - ...) by an ordered shuffle chain, so x is bitwise equal to the oracle
// and to the template-SELL kernels (G14).
template <int G, int R, bool LOWER>
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
    double acc = rhs[row];
    for (int64_t c = b0; c < b1; c += G) {
      const int64_t p = c + lane;
      const double pr = p < b1 ? __dmul_rn(vals[p], xo[P.ci[p]]) : 0.0;
      const int cnt = (int)min((int64_t)G, b1 - c);
      for (int q = 0; q < cnt; q++) acc = __dsub_rn(acc, tile.shfl(pr, q));
    }
    if (lane == 0) {
      double u = acc;
      if (!LOWER) u = __ddiv_rn(u, ud[row]);
      const double v =
          (omega == 1.0) ? u : __dadd_rn(__dmul_rn(1.0 - omega, xo[row]), __dmul_rn(omega, u));
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
  constexpr int R = 1;
  const int threads = 256, gpb = threads / G;
  int64_t blocks = (r1 - r0 + (int64_t)gpb * R - 1) / ((int64_t)gpb * R);
  if (blocks > (1ll << 30)) blocks = 1ll << 30;
#define FASTILU_JAC(GG)                                                                 \
  jacobi_kernel<GG, R, LOWER><<<(unsigned)blocks, threads, 0, st>>>(P, vals, ud, rhs, xo, xn, xf, \
                                                                      s, r0, r1, Gh, omega, final)
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

// ----------------------------------------------------------------------------------------
// Template-SELL kernels (one lane per row).  The template arrays are staged
// in shared memory; every value access is a coalesced 32-row slot, no index arrays are read.
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ bool tbit(const unsigned long long *m, int w) {
  return (m[w >> 6] >> (w & 63)) & 1ull;
}

// A's values in CSR order -> A's template slots (once per fastilu_set_values; lane per row).
__global__ void __launch_bounds__(256)
tsell_gather_a_kernel(TDev t, const double *__restrict__ aval, int64_t r0, int64_t nrows,
                      double *__restrict__ aT) {
  const int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  const int64_t sl = i >> 5, ln = i & 31;
  for (int a = 0; a < t.WA; a++) {
    const int32_t q = t.asrc[(sl * t.WA + a) * 32 + ln];
    aT[(sl * t.WA + a) * 32 + ln] = q >= 0 ? aval[q] : 0.0;
  }
}

// Multi-GPU factor halo on the template layout: only the columns [c0, W) of
// a ghost row -- its diagonal and strict-upper part -- are read by the sweep kernels (pivot rows
// u_kj, divisor u_jj), so the halo moves those, packed slice by slice: buf[(s NC + c) 32 + l] =
// vals[((slice0 + s) W + c0 + c) 32 + l], NC = W - c0 (coalesced both ways).
__global__ void tsell_pack_upper_kernel(const double *__restrict__ vals, int64_t slice0,
                                        int64_t total, int W, int c0, double *__restrict__ buf) {
  const int64_t per = (int64_t)(W - c0) * 32;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = q / per, rem = q - s * per;
    buf[q] = vals[(slice0 + s) * W * 32 + (int64_t)c0 * 32 + rem];
  }
}

// inverse of the pack into the ghost slices; column c0 also refreshes the compact diagonal copy
// (udiag, read by the register-pivot kernels)
__global__ void tsell_unpack_upper_kernel(const double *__restrict__ buf, int64_t slice0,
                                          int64_t total, int W, int c0, double *__restrict__ vals,
                                          double *__restrict__ udiag) {
  const int64_t per = (int64_t)(W - c0) * 32;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = q / per, rem = q - s * per;
    const double v = buf[q];
    vals[(slice0 + s) * W * 32 + (int64_t)c0 * 32 + rem] = v;
    if (rem < 32) udiag[(slice0 + s) * 32 + rem] = v;
  }
}

cudaError_t launch_tsell_pack_upper(const double *vals, int64_t slice0, int64_t nslices, int W,
                                    int c0, double *buf, cudaStream_t st) {
  const int64_t total = nslices * (int64_t)(W - c0) * 32;
  if (total <= 0) return cudaSuccess;
  tsell_pack_upper_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 4096), 256, 0, st>>>(
      vals, slice0, total, W, c0, buf);
  return cudaGetLastError();
}

cudaError_t launch_tsell_unpack_upper(const double *buf, int64_t slice0, int64_t nslices, int W,
                                      int c0, double *vals, double *udiag, cudaStream_t st) {
  const int64_t total = nslices * (int64_t)(W - c0) * 32;
  if (total <= 0) return cudaSuccess;
  tsell_unpack_upper_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 4096), 256, 0,
                              st>>>(buf, slice0, total, W, c0, vals, udiag);
  return cudaGetLastError();
}

cudaError_t launch_tsell_gather_a(const TDev &t, const double *aval, int64_t nrows, double *aT,
                                  cudaStream_t st) {
  return launch_tsell_gather_a_range(t, aval, 0, nrows, aT, st);
}

cudaError_t launch_tsell_gather_a_range(const TDev &t, const double *aval, int64_t r0,
                                        int64_t r1, double *aT, cudaStream_t st) {
  if (r1 <= r0) return cudaSuccess;
  tsell_gather_a_kernel<<<(unsigned)((r1 - r0 + 255) / 256), 256, 0, st>>>(t, aval, r0, r1, aT);
  return cudaGetLastError();
}

// a2/a3 on the template layout: ahat on A's sub-template and the initial guess (R4, R5).
// Reads A's values from their template copy aT (coalesced), writes ahatT and iterate 0.
__global__ void __launch_bounds__(256)
tsell_init_kernel(TDev t, const double *__restrict__ aT, const double *__restrict__ s,
                  const double *__restrict__ ad, int64_t r0, int64_t r1,
                  double *__restrict__ ahatT, double *__restrict__ vals,
                  double *__restrict__ udiag, ErrFlags *err, double shift, bool iter0) {
  __shared__ int32_t soff[128], soffA[128];
  __shared__ int8_t sw2a[128], sa2w[128];
  for (int q = threadIdx.x; q < t.W; q += blockDim.x) {
    soff[q] = t.off[q];
    sw2a[q] = t.w2a[q];
    if (t.w2a[q] >= 0) sa2w[t.w2a[q]] = (int8_t)q;
  }
  for (int q = threadIdx.x; q < t.WA; q += blockDim.x) soffA[q] = t.offA[q];
  __syncthreads();
  const int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r1) return;
  const int64_t sl = i >> 5, ln = i & 31;
  unsigned long long m[2] = {0ull, 0ull};
  for (int q = 0; q < t.words; q++) m[q] = t.mask[(sl * t.words + q) * 32 + ln];
  const double si = s[i];
  const double *arow = aT + sl * t.WA * 32 + ln;
  double *hrow = ahatT + sl * t.WA * 32 + ln;
  if (!iter0) {  // ahat only (the fused first sweep derives iterate 0 from it): A's columns
    for (int a = 0; a < t.WA; a++) {
      const int w = sa2w[a];
      double av = arow[a * 32];
      if (w == t.c0) av = __dadd_rn(av, __dmul_rn(shift, fabs(av)));
      const double ah = tbit(m, w) ? __dmul_rn(__dmul_rn(av, si), s[i + soffA[a]]) : 0.0;
      hrow[a * 32] = ah;
      if (w == t.c0 && bad_pivot(ah)) atomicMin(&err->zero_pivot, (unsigned long long)i);
    }
    return;
  }
  for (int w = 0; w < t.W; w++) {
    const int a = sw2a[w];
    double v = 0.0;  // fill entries and slots outside S: +0.0
    if (a >= 0) {
      // (a_ij s_i) s_j; A's absent template slots hold 0 and give +0 (never read as S entries)
      double av = arow[a * 32];
      if (w == t.c0) av = __dadd_rn(av, __dmul_rn(shift, fabs(av)));  // Manteuffel shift
      const double ah = tbit(m, w) ? __dmul_rn(__dmul_rn(av, si), s[i + soffA[a]]) : 0.0;
      hrow[a * 32] = ah;
      if (tbit(m, w)) v = (w < t.c0) ? __ddiv_rn(ah, ad[i + soff[w]]) : ah;
    }
    if (iter0) vals[(sl * t.W + w) * 32 + ln] = v;
    if (w == t.c0) {
      if (iter0) udiag[i] = v;
      if (bad_pivot(v)) atomicMin(&err->zero_pivot, (unsigned long long)i);
    }
  }
}

cudaError_t launch_tsell_init(const TDev &t, const double *aT, const double *s,
                              const double *ad, int64_t r0, int64_t r1, double *ahatT,
                              double *vals, double *udiag, ErrFlags *err, double shift,
                              cudaStream_t st, bool iter0) {
  if (r1 <= r0) return cudaSuccess;
  tsell_init_kernel<<<(unsigned)((r1 - r0 + 255) / 256), 256, 0, st>>>(
      t, aT, s, ad, r0, r1, ahatT, vals, udiag, err, shift, iter0);
  return cudaGetLastError();
}

// a8/a9 on the template layout: the oracle's row sums in the oracle's order (ascending
// columns, rounded product then difference), absent slots skipped => bitwise equal.
template <bool LOWER>
__global__ void __launch_bounds__(256)
tsell_jacobi_kernel(TDev t, const double *__restrict__ vals, const double *__restrict__ ud,
                    const double *__restrict__ rhs, const double *__restrict__ xo,
                    double *__restrict__ xn, double *__restrict__ xf,
                    const double *__restrict__ s, int64_t r0, int64_t r1, int64_t Gh,
                    double omega, bool final) {
  __shared__ int32_t soff[128];
  for (int q = threadIdx.x; q < t.W; q += blockDim.x) soff[q] = t.off[q];
  __syncthreads();
  const int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r1) return;
  const int64_t sl = i >> 5, ln = i & 31;
  unsigned long long m[2] = {0ull, 0ull};
  for (int q = 0; q < t.words; q++) m[q] = t.mask[(sl * t.words + q) * 32 + ln];
  const double *row = vals + sl * t.W * 32 + ln;
  double acc = rhs[i];
  const int w0 = LOWER ? 0 : t.c0 + 1, w1 = LOWER ? t.c0 : t.W;
  for (int w = w0; w < w1; w++)
    if (tbit(m, w)) acc = __dsub_rn(acc, __dmul_rn(row[w * 32], xo[i + soff[w]]));
  if (!LOWER) acc = __ddiv_rn(acc, ud[i]);
  const double v = (omega == 1.0) ? acc
                                  : __dadd_rn(__dmul_rn(1.0 - omega, xo[i]), __dmul_rn(omega, acc));
  if (final) xf[i - Gh] = __dmul_rn(s[i], v); else xn[i] = v;
}

cudaError_t launch_tsell_jacobi(const TDev &t, bool lower, const double *vals,
                                const double *udiag, const double *rhs, const double *xo,
                                double *xn, double *xfinal, const double *s, int64_t r0,
                                int64_t r1, int64_t Gh, double omega, bool final,
                                cudaStream_t st) {
  if (r1 <= r0) return cudaSuccess;
  const unsigned blocks = (unsigned)((r1 - r0 + 255) / 256);
  if (lower)
    tsell_jacobi_kernel<true><<<blocks, 256, 0, st>>>(t, vals, udiag, rhs, xo, xn, xfinal, s, r0,
                                                       r1, Gh, omega, final);
  else
    tsell_jacobi_kernel<false><<<blocks, 256, 0, st>>>(t, vals, udiag, rhs, xo, xn, xfinal, s,
                                                        r0, r1, Gh, omega, final);
  return cudaGetLastError();
}

__global__ void reduce_reset_kernel(const double *__restrict__ partials, int np, double *dst,
                                    unsigned int *counter) {
  __shared__ double sh[1024];
  double t = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) t += partials[i];
  sh[threadIdx.x] = t;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *dst = sh[0];
    if (counter) *counter = 0u;
  }
}

cudaError_t launch_reduce_reset(const double *partials, int np, double *dst,
                                unsigned int *counter, cudaStream_t st) {
  reduce_reset_kernel<<<1, 1024, 0, st>>>(partials, np, dst, counter);
  return cudaGetLastError();
}

__global__ void sumsq_kernel(const double *__restrict__ x, int64_t n, double *partials) {
  double t = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    t = fma(x[i], x[i], t);
  __shared__ double wsum[32];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double u = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) u += wsum[w];
    partials[blockIdx.x] = u;
  }
}

cudaError_t launch_sumsq(const double *x, int64_t n, double *partials, double *dst,
                         cudaStream_t st) {
  sumsq_kernel<<<kSumsqBlocks, 256, 0, st>>>(x, n, partials);
  reduce_kernel<<<1, 1024, 0, st>>>(partials, kSumsqBlocks, dst);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------------------
// GMRES building blocks (config 5).  Reductions are deterministic (fixed grid, fixed trees).
// ----------------------------------------------------------------------------------------
template <int G>
__global__ void __launch_bounds__(256)
spmv_kernel(const int64_t *__restrict__ arp, const int32_t *__restrict__ aci,
            const double *__restrict__ aval, const double *__restrict__ x,
            double *__restrict__ y, int64_t r0, int64_t r1, int64_t Gh) {
  auto tile = cg::tiled_partition<G>(cg::this_thread_block());
  const int gpb = blockDim.x / G;
  const int lane = tile.thread_rank();
  const int64_t stride = (int64_t)gridDim.x * gpb;
  for (int64_t row = r0 + (int64_t)blockIdx.x * gpb + threadIdx.x / G; row < r1; row += stride) {
    double sum = 0.0;
    for (int64_t q = arp[row] + lane; q < arp[row + 1]; q += G) sum = fma(aval[q], x[aci[q]], sum);
    sum = cg::reduce(tile, sum, cg::plus<double>());
    if (lane == 0) y[row - Gh] = sum;
  }
}

cudaError_t launch_spmv(const int64_t *arp, const int32_t *aci, const double *aval,
                        const double *x, double *y, int64_t r0, int64_t r1, int64_t Gh, int G,
                        cudaStream_t st) {
  if (r1 <= r0) return cudaSuccess;
  const int threads = 256, gpb = threads / G;
  int64_t blocks = (r1 - r0 + gpb - 1) / gpb;
  if (blocks > (1ll << 30)) blocks = 1ll << 30;
  switch (G) {
    case 4: spmv_kernel<4><<<(unsigned)blocks, threads, 0, st>>>(arp, aci, aval, x, y, r0, r1, Gh); break;
    case 8: spmv_kernel<8><<<(unsigned)blocks, threads, 0, st>>>(arp, aci, aval, x, y, r0, r1, Gh); break;
    case 16: spmv_kernel<16><<<(unsigned)blocks, threads, 0, st>>>(arp, aci, aval, x, y, r0, r1, Gh); break;
    default: spmv_kernel<32><<<(unsigned)blocks, threads, 0, st>>>(arp, aci, aval, x, y, r0, r1, Gh); break;
  }
  return cudaGetLastError();
}

// GMRES orthogonalisation (Sec. 7b), HBM-bound: every kernel reads each V_j it needs once.
// mdot: block b owns chunks of kChunk rows (kRpt rows per thread, 256-row stride); the chunk's w
// values stay in registers while the block walks j = 0..k-1 (one coalesced read of V_j per
// chunk), each warp reduces its V_j . w share by shuffles into its own shared-memory slot
// (fixed order: deterministic), and the block's k partials go to partials[j * grid + b].
constexpr int kRpt = 8, kChunk = 256 * kRpt, kMaxK = 128;
static unsigned orth_blocks(int64_t n) {
  const int64_t chunks = (n + kChunk - 1) / kChunk;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(chunks, kDotBlocks));
}

__global__ void __launch_bounds__(256)
mdot_kernel(const double *__restrict__ V, int64_t ldv, int k, const double *__restrict__ extra,
            const double *__restrict__ w, int64_t n, double *__restrict__ partials) {
  __shared__ double red[8][kMaxK];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = threadIdx.x; j < 8 * kMaxK; j += blockDim.x) (&red[0][0])[j] = 0.0;
  __syncthreads();
  for (int64_t c0 = (int64_t)blockIdx.x * kChunk; c0 < n; c0 += (int64_t)gridDim.x * kChunk) {
    double wv[kRpt];
#pragma unroll
    for (int r = 0; r < kRpt; r++) {
      const int64_t i = c0 + r * 256 + threadIdx.x;
      wv[r] = i < n ? w[i] : 0.0;
    }
#pragma unroll 2
    for (int j = 0; j < k; j++) {
      const double *vj = (extra && j == k - 1) ? extra : V + (int64_t)j * ldv;
      double a = 0.0;
#pragma unroll
      for (int r = 0; r < kRpt; r++) {
        const int64_t i = c0 + r * 256 + threadIdx.x;
        if (i < n) a = fma(vj[i], wv[r], a);
      }
      for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
      if (lane == 0) red[warp][j] += a;
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    double t = 0.0;
    for (int q = 0; q < 8; q++) t += red[q][j];
    partials[(int64_t)j * gridDim.x + blockIdx.x] = t;
  }
}

__global__ void mdot_reduce_kernel(const double *__restrict__ partials, int nb, int k,
                                   double *__restrict__ out) {
  __shared__ double sh[256];
  for (int j = blockIdx.x; j < k; j += gridDim.x) {
    double t = 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) t += partials[(int64_t)j * nb + b];
    sh[threadIdx.x] = t;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[j] = sh[0];
    __syncthreads();
  }
}

cudaError_t launch_mdot(const double *V, int64_t ldv, int k, const double *w, int64_t n,
                        double *partials, double *out, cudaStream_t st, const double *extra) {
  if (k <= 0) return cudaSuccess;
  const int kk = k + (extra ? 1 : 0);  // out[k] = extra . w
  if (kk > kMaxK) return cudaErrorInvalidValue;
  const unsigned nb = orth_blocks(n);
  mdot_kernel<<<nb, 256, 0, st>>>(V, ldv, kk, extra, w, n, partials);
  mdot_reduce_kernel<<<min(kk, 64), 256, 0, st>>>(partials, (int)nb, kk, out);
  return cudaGetLastError();
}

// w += sign-scaled V c over kRpt rows per thread (independent FMA chains, the loads of a column
// issued together): the GMRES solution update x = M^-1 (V y) and the explicit re-projection of a
// pending vector after a severe cancellation.
__global__ void __launch_bounds__(256)
maxpy_kernel(const double *__restrict__ V, int64_t ldv, int k, const double *__restrict__ c,
             double *__restrict__ w, int64_t n, double sign) {
  __shared__ double sc[kMaxK];
  for (int j = threadIdx.x; j < k && j < kMaxK; j += blockDim.x) sc[j] = sign * c[j];
  __syncthreads();
  for (int64_t c0 = (int64_t)blockIdx.x * kChunk; c0 < n; c0 += (int64_t)gridDim.x * kChunk) {
    double t[kRpt];
#pragma unroll
    for (int r = 0; r < kRpt; r++) {
      const int64_t i = c0 + r * 256 + threadIdx.x;
      t[r] = i < n ? w[i] : 0.0;
    }
#pragma unroll 4
    for (int j = 0; j < k; j++) {
      const double *vj = V + (int64_t)j * ldv;
      const double cj = sc[j];
#pragma unroll
      for (int r = 0; r < kRpt; r++) {
        const int64_t i = c0 + r * 256 + threadIdx.x;
        if (i < n) t[r] = fma(cj, vj[i], t[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < kRpt; r++) {
      const int64_t i = c0 + r * 256 + threadIdx.x;
      if (i < n) w[i] = t[r];
    }
  }
}

cudaError_t launch_maxpy(const double *V, int64_t ldv, int k, const double *c, double *w,
                         int64_t n, double sign, cudaStream_t st) {
  if (k <= 0) return cudaSuccess;
  if (k > kMaxK) return cudaErrorInvalidValue;
  maxpy_kernel<<<orth_blocks(n), 256, 0, st>>>(V, ldv, k, c, w, n, sign);
  return cudaGetLastError();
}

// ---- DCGS2: classical Gram-Schmidt with the reorthogonalisation delayed by one iteration
// (DESIGN.md Sec. 7b).  Two passes over V per Arnoldi step: the dots of the pending vector
// u = V_p and of w = B u against V_0..V_p in one pass, then one pass that finalises
// q_p = (u - Q s) / rho and forms the next pending vector (w - Q z - q_p c_p) / rho.
// Block b owns the contiguous rows [b n / grid, (b+1) n / grid) (equal shares), kDRpt rows per
// thread and chunk.
// one wave: SMs x resident blocks of `func` (at most kDotBlocks), fewer for short vectors
static unsigned dcgs_blocks(int64_t n, int rpt, const void *func) {
  int dev = 0, per_sm = 1;
  cudaGetDevice(&dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, func, 256, 0) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int64_t chunks = (n + 256 * rpt - 1) / (256 * rpt);
  const int64_t wave = std::min<int64_t>((int64_t)sm_count(dev) * per_sm, kDotBlocks);
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(chunks, wave));
}

// out (per block): partials[(2 j + e) * grid + b] = V_j . u (e = 0), V_j . w (e = 1), j <= p.
// Groups of 4 columns x 2 vectors = 8 per-lane sums are reduced across the warp by a butterfly
// (each step halves the values a lane carries: 4 + 2 + 1 + 2 shuffles for 8 sums instead of 40);
// lane 4 t then holds sum t, summed into the warp's shared-memory slot (fixed order:
// deterministic).  RPT rows per thread and chunk; PF: the next group's loads are issued before
// the current group's multiply-adds and butterfly.
template <int RPT, bool PF, int MINB>
__global__ void __launch_bounds__(256, MINB)
dcgs_dot_kernel(const double *__restrict__ V, int64_t ldv, int p, const double *__restrict__ w,
                int64_t n, double *__restrict__ partials) {
  __shared__ double red[8][2 * kMaxK];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, k = p + 1;
  for (int j = threadIdx.x; j < 8 * 2 * kMaxK; j += blockDim.x) (&red[0][0])[j] = 0.0;
  __syncthreads();
  const int64_t rb = n * (int64_t)blockIdx.x / gridDim.x;
  const int64_t re = n * (int64_t)(blockIdx.x + 1) / gridDim.x;
  const double *u = V + (int64_t)p * ldv;
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  const int slot = (lane >> 2) & 7;  // the sum lane 4 t ends up with: column t / 2, vector t % 2
  for (int64_t c0 = rb; c0 < re; c0 += 256 * RPT) {
    double uv[RPT], wv[RPT], v[4][RPT];
#pragma unroll
    for (int r = 0; r < RPT; r++) {
      const int64_t i = c0 + r * 256 + threadIdx.x;
      uv[r] = i < re ? u[i] : 0.0;
      wv[r] = (w && i < re) ? w[i] : 0.0;
    }
    auto load = [&](int j0, double (&d)[4][RPT]) {
#pragma unroll
      for (int t = 0; t < 4; t++) {
        const double *vj = V + (int64_t)(j0 + t) * ldv;
#pragma unroll
        for (int r = 0; r < RPT; r++) {
          const int64_t i = c0 + r * 256 + threadIdx.x;
          d[t][r] = (j0 + t < k && i < re) ? vj[i] : 0.0;
        }
      }
    };
    if (PF) load(0, v);
    for (int j0 = 0; j0 < k; j0 += 4) {
      double nx[4][RPT];
      if (PF) {
        if (j0 + 4 < k) load(j0 + 4, nx);
      } else {
        load(j0, v);
      }
      double a[8];
#pragma unroll
      for (int t = 0; t < 4; t++) {
        a[2 * t] = a[2 * t + 1] = 0.0;
#pragma unroll
        for (int r = 0; r < RPT; r++) {
          a[2 * t] = fma(v[t][r], uv[r], a[2 * t]);
          a[2 * t + 1] = fma(v[t][r], wv[r], a[2 * t + 1]);
        }
      }
#pragma unroll
      for (int t = 0; t < 4; t++)
        a[t] = (b4 ? a[4 + t] : a[t]) + __shfl_xor_sync(0xffffffffu, b4 ? a[t] : a[4 + t], 16);
#pragma unroll
      for (int t = 0; t < 2; t++)
        a[t] = (b3 ? a[2 + t] : a[t]) + __shfl_xor_sync(0xffffffffu, b3 ? a[t] : a[2 + t], 8);
      a[0] = (b2 ? a[1] : a[0]) + __shfl_xor_sync(0xffffffffu, b2 ? a[0] : a[1], 4);
      a[0] += __shfl_xor_sync(0xffffffffu, a[0], 2);
      a[0] += __shfl_xor_sync(0xffffffffu, a[0], 1);
      if ((lane & 3) == 0 && j0 + (slot >> 1) < k) red[warp][2 * j0 + slot] += a[0];
      if (PF) {
#pragma unroll
        for (int t = 0; t < 4; t++)
#pragma unroll
          for (int r = 0; r < RPT; r++) v[t][r] = nx[t][r];
      }
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < 2 * k; j += blockDim.x) {
    double t = 0.0;
    for (int q = 0; q < 8; q++) t += red[q][j];
    partials[(int64_t)j * gridDim.x + blockIdx.x] = t;
  }
}

template <int RPT, bool PF, int MINB>
static cudaError_t dcgs_dot_run(const double *V, int64_t ldv, int p, const double *w, int64_t n,
                                double *partials, double *out, cudaStream_t st) {
  const unsigned nb = dcgs_blocks(n, RPT, (const void *)dcgs_dot_kernel<RPT, PF, MINB>);
  dcgs_dot_kernel<RPT, PF, MINB><<<nb, 256, 0, st>>>(V, ldv, p, w, n, partials);
  mdot_reduce_kernel<<<min(2 * (p + 1), 64), 256, 0, st>>>(partials, (int)nb, 2 * (p + 1), out);
  return cudaGetLastError();
}

cudaError_t launch_dcgs_dot(const double *V, int64_t ldv, int p, const double *w, int64_t n,
                            double *partials, double *out, cudaStream_t st) {
  if (p < 0 || p + 1 > kMaxK) return cudaErrorInvalidValue;
  // measured (config 5, profiles/r2zd_dcgs_variants.log): 4 rows per thread without the
  // software prefetch is the fastest of the shapes tried (6.9 TB/s)
  return dcgs_dot_run<4, false, 3>(V, ldv, p, w, n, partials, out, st);
}

// coef = [s_0..s_{p-1}, z_0..z_{p-1}, c_p, 1/rho] (device):
//   q = (V_p - sum_j s_j V_j) / rho -> V_p;   (w - sum_j z_j V_j - c_p q) / rho -> V_{p+1}
// RPT rows per thread and chunk, UNR columns' loads in flight
template <int RPT, int UNR>
__global__ void __launch_bounds__(256)
dcgs_update_kernel(double *__restrict__ V, int64_t ldv, int p, const double *__restrict__ coef,
                   const double *__restrict__ w, int64_t n) {
  __shared__ double sc[2 * kMaxK + 2];
  for (int j = threadIdx.x; j < 2 * p + 2; j += blockDim.x) sc[j] = coef[j];
  __syncthreads();
  const double cp = sc[2 * p], irho = sc[2 * p + 1];
  const int64_t rb = n * (int64_t)blockIdx.x / gridDim.x;
  const int64_t re = n * (int64_t)(blockIdx.x + 1) / gridDim.x;
  double *u = V + (int64_t)p * ldv, *un = u + ldv;
  for (int64_t c0 = rb; c0 < re; c0 += 256 * RPT) {
    double t1[RPT], t2[RPT];
#pragma unroll
    for (int r = 0; r < RPT; r++) {
      const int64_t i = c0 + r * 256 + threadIdx.x;
      t1[r] = i < re ? u[i] : 0.0;
      t2[r] = i < re ? w[i] : 0.0;
    }
#pragma unroll UNR
    for (int j = 0; j < p; j++) {
      const double *vj = V + (int64_t)j * ldv;
      const double sj = sc[j], zj = sc[p + j];
#pragma unroll
      for (int r = 0; r < RPT; r++) {
        const int64_t i = c0 + r * 256 + threadIdx.x;
        const double v = i < re ? vj[i] : 0.0;
        t1[r] = fma(-sj, v, t1[r]);
        t2[r] = fma(-zj, v, t2[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < RPT; r++) {
      const int64_t i = c0 + r * 256 + threadIdx.x;
      if (i < re) {
        const double q = t1[r] * irho;
        u[i] = q;
        un[i] = fma(-cp, q, t2[r]) * irho;
      }
    }
  }
}

template <int RPT, int UNR>
static cudaError_t dcgs_update_run(double *V, int64_t ldv, int p, const double *coef,
                                   const double *w, int64_t n, cudaStream_t st) {
  dcgs_update_kernel<RPT, UNR>
      <<<dcgs_blocks(n, RPT, (const void *)dcgs_update_kernel<RPT, UNR>), 256, 0, st>>>(
          V, ldv, p, coef, w, n);
  return cudaGetLastError();
}

cudaError_t launch_dcgs_update(double *V, int64_t ldv, int p, const double *coef, const double *w,
                               int64_t n, cudaStream_t st) {
  if (p < 0 || p + 1 > kMaxK) return cudaErrorInvalidValue;
  if (n <= 0) return cudaSuccess;
  return dcgs_update_run<4, 4>(V, ldv, p, coef, w, n, st);  // 5.9 TB/s; see dcgs_dot
}

__global__ void axpby_kernel(double a, const double *__restrict__ x, double b,
                             double *__restrict__ y, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (b == 0.0) ? a * x[i] : fma(a, x[i], b * y[i]);
}

cudaError_t launch_axpby(double a, const double *x, double b, double *y, int64_t n,
                         cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  axpby_kernel<<<vec_blocks(n), 256, 0, st>>>(a, x, b, y, n);
  return cudaGetLastError();
}


}  // namespace fastilu
