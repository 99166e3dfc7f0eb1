// Block (BSR) sweep for patterns made of dense BS x BS blocks: the 3-dof "elasticity" patterns
// of the paper's own experiments (Table 6: 3-dof 27-point, ILU(3)), SURVEY.md
// Sec. 8(f) item 4 ("3x3-block-vectorised kernels").
//
// S is block-dense for these matrices (every scalar level is uniform over a node block, checked
// on the host at create time), so the scalar synchronous sweep (readings R1-R3)
// regroups exactly into block terms: for target entry (i, j) = (BS I + d, BS J + e),
//
//   acc = ahat_ij - sum_{K < min(I,J), (I,K),(K,J) in S}  sum_{c=0..BS-1} l_{i,BS K+c} u_{BS K+c,j}
//                 - sum_{c < (j < i ? e : d) restricted to k < min(i,j)} (tail inside block min(I,J))
//
// with k = BS K + c ascending, i.e. the oracle's order (ascending pivots, rounded product then
// rounded difference), so the result is bitwise the scalar sweep's.  The pivot-block pairs
// (I,K),(K,J) of every target block are listed once on the host (ascending K); one thread owns
// one target block: 9 accumulators in registers, no index matching and no synchronisation on
// the device.  Blocks are stored contiguously, BS*BS values padded to an even count (16-byte
// aligned vector loads).
#include <algorithm>

#include "device.h"

namespace fastilu {

static __device__ __forceinline__ bool bsr_bad_pivot(double d) {
  return !(d != 0.0 && isfinite(d));
}

template <int BB, int ST>
static __device__ __forceinline__ void ld_block(const double *__restrict__ p, double (&v)[BB]) {
  const double2 *q = reinterpret_cast<const double2 *>(p);
#pragma unroll
  for (int h = 0; h < ST / 2; h++) {
    const double2 x = __ldg(q + h);
    v[2 * h] = x.x;
    if (2 * h + 1 < BB) v[2 * h + 1] = x.y;
  }
}

// generic address (shared-memory stage or global)
template <int BB, int ST>
static __device__ __forceinline__ void ld_block_any(const double *p, double (&v)[BB]) {
  const double2 *q = reinterpret_cast<const double2 *>(p);
#pragma unroll
  for (int h = 0; h < ST / 2; h++) {
    const double2 x = q[h];
    v[2 * h] = x.x;
    if (2 * h + 1 < BB) v[2 * h + 1] = x.y;
  }
}

template <int BB, int ST>
static __device__ __forceinline__ void st_block(double *__restrict__ p, const double (&v)[BB]) {
  double2 *q = reinterpret_cast<double2 *>(p);
#pragma unroll
  for (int h = 0; h < ST / 2; h++) q[h] = make_double2(v[2 * h], 2 * h + 1 < BB ? v[2 * h + 1] : 0.0);
}

// The within-block tail terms and the update of target block b = (I, J) after its pivot-block
// terms (accumulators a), shared by the block sweeps: L blocks divide by the old diagonal block
// of row J, the diagonal block finishes its own LU, U blocks use the L part of row I's diagonal
// block; residual defects into r2; the new block is stored to out.  lbase: where the tile's own
// blocks are read (a shared-memory stage or `old`).
template <int BS>
static __device__ __forceinline__ void bsr_finish(const BsrDev &B, int64_t b, int I, int J,
                                                  double (&a)[BS * BS], const double *lbase,
                                                  const double *__restrict__ old,
                                                  double *__restrict__ out, double omega,
                                                  double &r2, ErrFlags *err) {
  constexpr int BB = BS * BS, ST = (BB + 1) & ~1;
  const bool damp = (omega != 1.0);
  const double om1 = 1.0 - omega;
    double o[BB], nv[BB];
    ld_block_any<BB, ST>(lbase + b * ST, o);
    if (J < I) {  // L block: tail k = BS J + c, c < e; divide by u_jj of iterate s-1 (R1)
      double D[BB];
      ld_block<BB, ST>(old + (int64_t)B.bdiag[J] * ST, D);
#pragma unroll
      for (int d = 0; d < BS; d++)
#pragma unroll
        for (int e = 0; e < BS; e++) {
          double v = a[d * BS + e];
#pragma unroll
          for (int c = 0; c < e; c++) v = __dsub_rn(v, __dmul_rn(o[d * BS + c], D[c * BS + e]));
          const double ujj = D[e * BS + e], ol = o[d * BS + e];
          const double ee = __dsub_rn(v, __dmul_rn(ol, ujj));
          r2 = fma(ee, ee, r2);
          const double l = __ddiv_rn(v, ujj);
          nv[d * BS + e] = damp ? __dadd_rn(__dmul_rn(om1, ol), __dmul_rn(omega, l)) : l;
        }
    } else if (J == I) {  // diagonal block: tail c < min(d, e)
#pragma unroll
      for (int d = 0; d < BS; d++)
#pragma unroll
        for (int e = 0; e < BS; e++) {
          double v = a[d * BS + e];
#pragma unroll
          for (int c = 0; c < (d < e ? d : e); c++)
            v = __dsub_rn(v, __dmul_rn(o[d * BS + c], o[c * BS + e]));
          const double od = o[d * BS + e];
          if (d > e) {
            const double ujj = o[e * BS + e];
            const double ee = __dsub_rn(v, __dmul_rn(od, ujj));
            r2 = fma(ee, ee, r2);
            const double l = __ddiv_rn(v, ujj);
            nv[d * BS + e] = damp ? __dadd_rn(__dmul_rn(om1, od), __dmul_rn(omega, l)) : l;
          } else {
            const double ee = __dsub_rn(v, od);
            r2 = fma(ee, ee, r2);
            nv[d * BS + e] = damp ? __dadd_rn(__dmul_rn(om1, od), __dmul_rn(omega, v)) : v;
          }
        }
#pragma unroll
      for (int d = 0; d < BS; d++)
        if (bsr_bad_pivot(nv[d * BS + d]))
          atomicMin(&err->zero_pivot, (unsigned long long)I * BS + d);
    } else {  // U block: tail k = BS I + c, c < d, with the L part of the own diagonal block
      double D[BB];
      ld_block_any<BB, ST>(lbase + (int64_t)B.bdiag[I] * ST, D);
#pragma unroll
      for (int d = 0; d < BS; d++)
#pragma unroll
        for (int e = 0; e < BS; e++) {
          double v = a[d * BS + e];
#pragma unroll
          for (int c = 0; c < d; c++) v = __dsub_rn(v, __dmul_rn(D[d * BS + c], o[c * BS + e]));
          const double ou = o[d * BS + e];
          const double ee = __dsub_rn(v, ou);
          r2 = fma(ee, ee, r2);
          nv[d * BS + e] = damp ? __dadd_rn(__dmul_rn(om1, ou), __dmul_rn(omega, v)) : v;
        }
    }
    st_block<BB, ST>(out + b * ST, nv);
}

// One CTA takes tiles of blockDim.x consecutive target blocks (grid-stride over tiles).  With
// STAGE, the tile's block rows (all their blocks, iterate s-1) are first copied to shared memory
// when they fit in smem_blocks: the L blocks (I,K) every target of row I reads, the target's own
// old block and the row's diagonal block then come from shared memory; only the pivots' U blocks
// (K,J) and the divisor blocks of rows J are read from global memory.
template <int BS, bool STAGE, int MINB>
__global__ void __launch_bounds__(256, MINB)
bsr_sweep_kernel(BsrDev B, const double *__restrict__ ahb, const double *__restrict__ old,
                 double *__restrict__ out, double omega, double *__restrict__ partials,
                 ErrFlags *err, int smem_blocks) {
  constexpr int BB = BS * BS, ST = (BB + 1) & ~1;
  extern __shared__ __align__(16) double sblk[];
  double r2 = 0.0;
  const int64_t ntiles = (B.nblk + blockDim.x - 1) / blockDim.x;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t b = tile * blockDim.x + threadIdx.x;
    int64_t s0 = 0;
    bool staged = false;
    if (STAGE) {
      const int64_t bf = tile * blockDim.x;
      const int64_t bl = min(bf + (int64_t)blockDim.x, B.nblk) - 1;
      s0 = B.bptr[B.brow[bf]];
      const int64_t s1 = B.bptr[B.brow[bl] + 1];
      staged = (s1 - s0) <= smem_blocks;  // uniform over the CTA
      __syncthreads();                    // the previous tile's readers are done
      if (staged) {
        const double2 *src = reinterpret_cast<const double2 *>(old + s0 * ST);
        double2 *dst = reinterpret_cast<double2 *>(sblk);
        for (int64_t q = threadIdx.x; q < (s1 - s0) * (ST / 2); q += blockDim.x) dst[q] = src[q];
      }
      __syncthreads();
    }
    if (b >= B.nblk) continue;
    const double *lbase = staged ? sblk - s0 * ST : old;  // blocks of the tile's rows
    const int I = B.brow[b], J = B.bcol[b];
    double a[BB];
    ld_block<BB, ST>(ahb + b * ST, a);  // +0.0 for fill entries (R4)
    const int64_t t1 = B.tptr[b + 1];
    for (int64_t t = B.tptr[b]; t < t1; t++) {  // pivot blocks K ascending
      const int2 pr = B.terms[t];
      double L[BB], U[BB];
      ld_block_any<BB, ST>(lbase + (int64_t)pr.x * ST, L);
      ld_block<BB, ST>(old + (int64_t)pr.y * ST, U);
#pragma unroll
      for (int d = 0; d < BS; d++)
#pragma unroll
        for (int e = 0; e < BS; e++) {
          double v = a[d * BS + e];
#pragma unroll
          for (int c = 0; c < BS; c++) v = __dsub_rn(v, __dmul_rn(L[d * BS + c], U[c * BS + e]));
          a[d * BS + e] = v;
        }
    }
    bsr_finish<BS>(B, b, I, J, a, lbase, old, out, omega, r2, err);
  }
  // deterministic block reduction (fixed shuffle tree, then warps in order)
  __shared__ double wsum[32];
  double v = r2;
  for (int q = 16; q > 0; q >>= 1) v += __shfl_down_sync(0xffffffffu, v, q);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += wsum[w];
    partials[blockIdx.x] = t;
  }
}

// The paper's ASYNCHRONOUS in-place sweep on the block layout ("updated in
// parallel (in place) ... non-deterministic"; option "Block Size (number of nonzeroes per
// thread)").  Thread q updates the nb consecutive target blocks [q nb, (q+1) nb)
// (block row order) one after the other, in place: every value it reads (pivot blocks, divisor
// blocks, its own earlier blocks) is whatever the factor holds at that moment, so entries it
// updated before are used fresh, entries of other threads maybe; inside a block the entries are
// updated in row-major order and the tail terms use the block's new values (Gauss-Seidel order).
// nb * BS^2 = nonzeros per thread.  The residual partials use the values the update read.
template <int BS>
__global__ void __launch_bounds__(256)
bsr_sweep_async_kernel(BsrDev B, const double *__restrict__ ahb, double *vals, double omega,
                       double *__restrict__ partials, ErrFlags *err, int nb) {
  constexpr int BB = BS * BS, ST = (BB + 1) & ~1;
  const bool damp = (omega != 1.0);
  const double om1 = 1.0 - omega;
  double r2 = 0.0;
  const int64_t nthr = (B.nblk + nb - 1) / nb;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nthr;
       q += (int64_t)gridDim.x * blockDim.x) {
    for (int64_t b = q * nb; b < min((q + 1) * (int64_t)nb, B.nblk); b++) {
      const int I = B.brow[b], J = B.bcol[b];
      double a[BB];
      ld_block<BB, ST>(ahb + b * ST, a);
      for (int64_t t = B.tptr[b]; t < B.tptr[b + 1]; t++) {  // pivot blocks K ascending
        const int2 pr = B.terms[t];
        double L[BB], U[BB];
        ld_block_any<BB, ST>(vals + (int64_t)pr.x * ST, L);
        ld_block_any<BB, ST>(vals + (int64_t)pr.y * ST, U);
#pragma unroll
        for (int d = 0; d < BS; d++)
#pragma unroll
          for (int e = 0; e < BS; e++) {
            double v = a[d * BS + e];
#pragma unroll
            for (int c = 0; c < BS; c++) v = __dsub_rn(v, __dmul_rn(L[d * BS + c], U[c * BS + e]));
            a[d * BS + e] = v;
          }
      }
      double o[BB], nv[BB];
      ld_block_any<BB, ST>(vals + b * ST, o);
      if (J < I) {
        double D[BB];
        ld_block_any<BB, ST>(vals + (int64_t)B.bdiag[J] * ST, D);
#pragma unroll
        for (int d = 0; d < BS; d++)
#pragma unroll
          for (int e = 0; e < BS; e++) {
            double v = a[d * BS + e];
#pragma unroll
            for (int c = 0; c < e; c++) v = __dsub_rn(v, __dmul_rn(nv[d * BS + c], D[c * BS + e]));
            const double ujj = D[e * BS + e], ol = o[d * BS + e];
            const double ee = __dsub_rn(v, __dmul_rn(ol, ujj));
            r2 = fma(ee, ee, r2);
            const double l = __ddiv_rn(v, ujj);
            nv[d * BS + e] = damp ? __dadd_rn(__dmul_rn(om1, ol), __dmul_rn(omega, l)) : l;
          }
      } else if (J == I) {
#pragma unroll
        for (int d = 0; d < BS; d++)
#pragma unroll
          for (int e = 0; e < BS; e++) {
            double v = a[d * BS + e];
#pragma unroll
            for (int c = 0; c < (d < e ? d : e); c++)
              v = __dsub_rn(v, __dmul_rn(nv[d * BS + c], nv[c * BS + e]));
            const double od = o[d * BS + e];
            if (d > e) {
              const double ujj = nv[e * BS + e];
              const double ee = __dsub_rn(v, __dmul_rn(od, ujj));
              r2 = fma(ee, ee, r2);
              const double l = __ddiv_rn(v, ujj);
              nv[d * BS + e] = damp ? __dadd_rn(__dmul_rn(om1, od), __dmul_rn(omega, l)) : l;
            } else {
              const double ee = __dsub_rn(v, od);
              r2 = fma(ee, ee, r2);
              nv[d * BS + e] = damp ? __dadd_rn(__dmul_rn(om1, od), __dmul_rn(omega, v)) : v;
            }
          }
#pragma unroll
        for (int d = 0; d < BS; d++)
          if (bsr_bad_pivot(nv[d * BS + d]))
            atomicMin(&err->zero_pivot, (unsigned long long)I * BS + d);
      } else {
        double D[BB];
        ld_block_any<BB, ST>(vals + (int64_t)B.bdiag[I] * ST, D);
#pragma unroll
        for (int d = 0; d < BS; d++)
#pragma unroll
          for (int e = 0; e < BS; e++) {
            double v = a[d * BS + e];
#pragma unroll
            for (int c = 0; c < d; c++) v = __dsub_rn(v, __dmul_rn(D[d * BS + c], nv[c * BS + e]));
            const double ou = o[d * BS + e];
            const double ee = __dsub_rn(v, ou);
            r2 = fma(ee, ee, r2);
            nv[d * BS + e] = damp ? __dadd_rn(__dmul_rn(om1, ou), __dmul_rn(omega, v)) : v;
          }
      }
      st_block<BB, ST>(vals + b * ST, nv);
    }
  }
  __shared__ double wsum[32];
  double v = r2;
  for (int q = 16; q > 0; q >>= 1) v += __shfl_down_sync(0xffffffffu, v, q);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += wsum[w];
    partials[blockIdx.x] = t;
  }
}

// scalar CSR (S row order) <-> block layout; one warp per scalar row r = BS I + d, whose S row
// is block row I's columns expanded (entry q of the row = block q / BS, column e = q % BS).
template <int BS, int DIR>  // DIR 0: CSR -> blocks, 1: blocks -> CSR (+ u_ii copy)
__global__ void bsr_convert_kernel(BsrDev B, const int64_t *__restrict__ rp,
                                   const double *__restrict__ src, double *__restrict__ dst,
                                   double *__restrict__ ud, int64_t nrows) {
  constexpr int ST = (BS * BS + 1) & ~1;
  const int lane = threadIdx.x & 31;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nrows;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t I = r / BS, d = r % BS, b0 = B.bptr[I], p0 = rp[r];
    const int m = (int)(rp[r + 1] - p0);
    for (int q = lane; q < m; q += 32) {
      const int64_t slot = (b0 + q / BS) * ST + d * BS + q % BS;
      if (DIR == 0) dst[slot] = src[p0 + q];
      else dst[p0 + q] = src[slot];
    }
    if (DIR == 1 && lane == 0) ud[r] = src[(int64_t)B.bdiag[I] * ST + d * BS + d];
  }
}

// ahat on A's pattern -> block layout (A entry q of row r sits at offset apos[q] of S row r)
template <int BS>
__global__ void bsr_ahat_kernel(BsrDev B, const int64_t *__restrict__ arp,
                                const int32_t *__restrict__ apos, const double *__restrict__ ahatA,
                                double *__restrict__ ahb, int64_t nrows) {
  constexpr int ST = (BS * BS + 1) & ~1;
  const int lane = threadIdx.x & 31;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nrows;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t I = r / BS, d = r % BS, b0 = B.bptr[I];
    for (int64_t q = arp[r] + lane; q < arp[r + 1]; q += 32) {
      const int p = apos[q];
      ahb[(b0 + p / BS) * ST + d * BS + p % BS] = ahatA[q];
    }
  }
}

#define FASTILU_BS_DISPATCH(BSV, CALL) \
  switch (BSV) {                       \
    case 2: { constexpr int BS = 2; CALL; } break; \
    case 3: { constexpr int BS = 3; CALL; } break; \
    case 4: { constexpr int BS = 4; CALL; } break; \
    default: return cudaErrorInvalidValue;         \
  }

template <int BS, int MINB>
static cudaError_t bsr_occ_t(int threads, size_t smem, int *bps) {
  auto k = smem ? bsr_sweep_kernel<BS, true, MINB> : bsr_sweep_kernel<BS, false, MINB>;
  if (smem) {
    cudaError_t e = allow_dynamic_smem((const void *)k);
    if (e != cudaSuccess) return e;
  }
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, k, threads, smem);
}

// MINB: resident-CTA hint (__launch_bounds__ min blocks): 1 = registers unconstrained, 4 = at
// most 64 registers (4 x 256 threads per SM)
cudaError_t bsr_sweep_occupancy(int bs, int threads, size_t smem, int minb, int *blocks_per_sm) {
  if (minb >= 4) {
    FASTILU_BS_DISPATCH(bs, return (bsr_occ_t<BS, 4>(threads, smem, blocks_per_sm)))
  } else {
    FASTILU_BS_DISPATCH(bs, return (bsr_occ_t<BS, 1>(threads, smem, blocks_per_sm)))
  }
  return cudaSuccess;
}

int bsr_block_stride(int bs) { return (bs * bs + 1) & ~1; }

template <int MINB>
static cudaError_t launch_bsr_t(const BsrDev &B, const double *ahb, const double *old,
                                double *out, double omega, double *partials, ErrFlags *err,
                                int grid, int threads, size_t smem, cudaStream_t st) {
  const int sb = smem ? (int)(smem / (8 * bsr_block_stride(B.bs))) : 0;
  if (smem) {
    FASTILU_BS_DISPATCH(B.bs, (bsr_sweep_kernel<BS, true, MINB><<<grid, threads, smem, st>>>(
                                  B, ahb, old, out, omega, partials, err, sb)))
  } else {
    FASTILU_BS_DISPATCH(B.bs, (bsr_sweep_kernel<BS, false, MINB><<<grid, threads, 0, st>>>(
                                  B, ahb, old, out, omega, partials, err, 0)))
  }
  return cudaGetLastError();
}

cudaError_t launch_bsr_sweep(const BsrDev &B, const double *ahb, const double *old, double *out,
                             double omega, double *partials, ErrFlags *err, int grid,
                             int threads, size_t smem, int minb, cudaStream_t st) {
  return minb >= 4 ? launch_bsr_t<4>(B, ahb, old, out, omega, partials, err, grid, threads, smem, st)
                   : launch_bsr_t<1>(B, ahb, old, out, omega, partials, err, grid, threads, smem, st);
}

cudaError_t launch_bsr_sweep_async(const BsrDev &B, const double *ahb, double *vals, double omega,
                                   double *partials, ErrFlags *err, int grid, int nb,
                                   cudaStream_t st) {
  FASTILU_BS_DISPATCH(B.bs, (bsr_sweep_async_kernel<BS><<<grid, 256, 0, st>>>(
                                B, ahb, vals, omega, partials, err, nb)))
  return cudaGetLastError();
}

static unsigned conv_grid(int64_t nrows) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((nrows + 7) / 8, 65535 * 16));
}

cudaError_t launch_bsr_from_csr(const BsrDev &B, const int64_t *rp, const double *vals,
                                double *vb, int64_t nrows, cudaStream_t st) {
  FASTILU_BS_DISPATCH(B.bs, (bsr_convert_kernel<BS, 0><<<conv_grid(nrows), 256, 0, st>>>(
                                B, rp, vals, vb, nullptr, nrows)))
  return cudaGetLastError();
}

cudaError_t launch_bsr_to_csr(const BsrDev &B, const int64_t *rp, const double *vb, double *vals,
                              double *ud, int64_t nrows, cudaStream_t st) {
  FASTILU_BS_DISPATCH(B.bs, (bsr_convert_kernel<BS, 1><<<conv_grid(nrows), 256, 0, st>>>(
                                B, rp, vb, vals, ud, nrows)))
  return cudaGetLastError();
}

cudaError_t launch_bsr_ahat(const BsrDev &B, const int64_t *arp, const int32_t *apos,
                            const double *ahatA, double *ahb, int64_t nrows, cudaStream_t st) {
  FASTILU_BS_DISPATCH(B.bs, (bsr_ahat_kernel<BS><<<conv_grid(nrows), 256, 0, st>>>(
                                B, arp, apos, ahatA, ahb, nrows)))
  return cudaGetLastError();
}

}  // namespace fastilu
