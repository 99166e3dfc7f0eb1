// L2 -> SM bandwidth microbenchmark (B200): every CTA streams chunks of an L2-resident buffer
// into shared memory with cp.async.bulk (TMA, mbarrier completion) or reads it with 128-bit
// loads; prints the achieved GB/s.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 l2bw.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mbar_init(unsigned a, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned ph) {
  unsigned d;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(d) : "r"(a), "r"(ph) : "memory");
  } while (!d);
}

template <int CHUNK, int NS>
__global__ void tma_kernel(const char *src, size_t span, int iters, unsigned long long *sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) unsigned long long bar[NS];
  const unsigned b0 = (unsigned)__cvta_generic_to_shared(bar), s0 = (unsigned)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    for (int q = 0; q < NS; q++) mbar_init(b0 + 8 * q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long acc = 0;
  const size_t nchunks = span / CHUNK;
  for (int it = 0; it < iters; it++) {
    const int st = it % NS;
    const unsigned ph = (it / NS) & 1;
    if (threadIdx.x == 0) {
      const size_t c = ((size_t)blockIdx.x * 7919 + (size_t)it * 104729) % nchunks;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b0 + 8 * st), "r"(CHUNK) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(s0 + st * CHUNK), "l"(src + c * CHUNK), "r"(CHUNK), "r"(b0 + 8 * st) : "memory");
    }
    mbar_wait(b0 + 8 * st, ph);
    acc += sm[st * CHUNK + threadIdx.x * 8];
    __syncthreads();
  }
  if (acc == 0x1234567) sink[0] = acc;
}

__global__ void ldg_kernel(const double2 *src, size_t n2, int iters, unsigned long long *sink) {
  double acc = 0;
  for (int it = 0; it < iters; it++) {
    const size_t base = (((size_t)blockIdx.x * 7919 + (size_t)it * 104729) * 4096) % (n2 - 4096);
    for (int k = threadIdx.x; k < 4096; k += blockDim.x) {
      const double2 v = src[base + k];
      acc += v.x + v.y;
    }
  }
  if (acc == 1.2345) sink[0] = 1;
}

int main() {
  const size_t span = 48ull << 20;  // 48 MB: L2-resident
  char *buf;
  unsigned long long *sink;
  cudaMalloc(&buf, span);
  cudaMemset(buf, 1, span);
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run_tma = [&](auto kern, int chunk, int ns, int blocks_per_sm) {
    const int smem = chunk * ns;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    kern<<<sms * blocks_per_sm, 128, smem>>>(buf, span, 10, sink);
    cudaEventRecord(a);
    kern<<<sms * blocks_per_sm, 128, smem>>>(buf, span, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("TMA bulk chunk=%6d stages=%d ctas/SM=%d: %8.1f GB/s  (%s)\n", chunk, ns, blocks_per_sm,
           (double)sms * blocks_per_sm * iters * chunk / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  run_tma(tma_kernel<16384, 2>, 16384, 2, 1);
  run_tma(tma_kernel<32768, 2>, 32768, 2, 1);
  run_tma(tma_kernel<32768, 3>, 32768, 3, 2);
  run_tma(tma_kernel<65536, 2>, 65536, 2, 1);
  run_tma(tma_kernel<65536, 3>, 65536, 3, 1);
  run_tma(tma_kernel<16384, 4>, 16384, 4, 2);
  for (int bps : {1, 2, 4}) {
    const int iters = 200;
    ldg_kernel<<<sms * bps, 512>>>((const double2 *)buf, span / 16, 5, sink);
    cudaEventRecord(a);
    ldg_kernel<<<sms * bps, 512>>>((const double2 *)buf, span / 16, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("LDG.128 512 thr x %d blocks/SM: %8.1f GB/s\n", bps,
           (double)sms * bps * iters * 4096 * 16 / ms / 1e6);
  }
  return 0;
}
