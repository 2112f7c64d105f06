// Microbenchmark: HBM streaming throughput of 1-D bulk copies (TMA engine) into an S-stage smem ring,
// one producer lane + one consumer warp per CTA, as a function of bytes in flight per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#ifndef NPROD
#define NPROD 1
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t x) { asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(x) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t p) {
#if defined(TEST_WAIT)
  asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.test_wait.parity.acquire.cta.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}\n" ::"r"(smem_u32(b)), "r"(p) : "memory");
#elif defined(HINT)
  asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 q, [%0], %1, %2;\n@!q bra W_%=;\n}\n" ::"r"(smem_u32(b)), "r"(p), "r"(HINT) : "memory");
#else
  asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}\n" ::"r"(smem_u32(b)), "r"(p) : "memory");
#endif
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
#ifdef CTA_FORM
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(d)), "l"(s), "r"(n), "r"(smem_u32(b)) : "memory");
#else
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(d)), "l"(s), "r"(n), "r"(smem_u32(b)) : "memory");
#endif
}

__global__ void stream_kernel(const uint8_t* src, size_t blocks_per_cta, int S, int blk, int copies, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = (uint64_t*)(smem + (size_t)S * blk);
  uint64_t* empty = full + S;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint8_t* base = src + (size_t)blockIdx.x * blocks_per_cta * blk;
  if (threadIdx.x >= 32 && threadIdx.x < 32 + NPROD) {
    for (size_t j = threadIdx.x - 32; j < blocks_per_cta; j += NPROD) {
      int st = j % S;
      if (j >= (size_t)S) mbar_wait(&empty[st], ((j / S) - 1) & 1);
      mbar_expect(&full[st], blk);
      for (int c = 0; c < copies; ++c) bulk(smem + (size_t)st * blk + c * (blk / copies), base + j * blk + c * (blk / copies), blk / copies, &full[st]);
    }
  } else if (threadIdx.x < 32) {
    float acc = 0.f;
    for (size_t j = 0; j < blocks_per_cta; ++j) {
      int st = j % S;
      mbar_wait(&full[st], (j / S) & 1);
      acc += (float)smem[(size_t)st * blk + threadIdx.x];
      __syncwarp();
      if (threadIdx.x == 0) mbar_arrive(&empty[st]);
    }
    if (acc == 1234.5f) sink[0] = acc;
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t total = (size_t)4 << 30;
  uint8_t* src; cudaMalloc(&src, total); cudaMemset(src, 1, total);
  float* sink; cudaMalloc(&sink, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct Cfg { int S, blk, copies, ctas_per_sm; };
  Cfg cfgs[] = {{15, 8192, 2, 1}, {24, 8192, 2, 1}, {26, 8192, 2, 1}, {8, 8192, 2, 2}, {12, 8192, 2, 2}, {30, 4096, 1, 1},
                {48, 4096, 1, 1}, {13, 16384, 4, 1}, {6, 32768, 8, 1}, {6, 32768, 1, 1}};
  for (auto c : cfgs) {
    int grid = sms * c.ctas_per_sm;
    size_t bpc = total / c.blk / grid;
    size_t smem = (size_t)c.S * c.blk + 2 * c.S * 8;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    stream_kernel<<<grid, 64, smem>>>(src, bpc, c.S, c.blk, c.copies, sink);
    cudaEventRecord(e0);
    stream_kernel<<<grid, 64, smem>>>(src, bpc, c.S, c.blk, c.copies, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("stages=%2d blk=%5d copies=%d ctas/SM=%d in-flight/SM=%4zu KB : %7.1f GB/s  (%s)\n", c.S, c.blk, c.copies,
           c.ctas_per_sm, smem * c.ctas_per_sm / 1024, (double)bpc * grid * c.blk / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
