// Decode-like streaming: NPROD producer lanes (lane l owns stage l), 8 KiB stages = K 4 KiB + V 4 KiB
// page-head blocks ([page][8 heads][4 KiB] layout), NCONS consumer warps taking every NCONS-th page.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t x) { asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(x) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t p) {
  asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}\n" ::"r"(smem_u32(b)), "r"(p) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(d)), "l"(s), "r"(n), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ int ldv(const int* p) { int v; asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory"); return v; }
__device__ __forceinline__ void stv(int* p, int v) { asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory"); }

constexpr int S = 15;
__global__ void k(const uint8_t* kp, const uint8_t* vp, int pages_per_cta, int nprod, int ncons, int heads, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = (uint64_t*)(smem + S * 8192);
  uint64_t* empty = full + S;
  int* tag = (int*)(empty + S);
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x < S) tag[threadIdx.x] = -1;
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); } asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  const int head = blockIdx.x % heads;
  const size_t page0 = (size_t)(blockIdx.x / heads) * pages_per_cta;
  if (warp == ncons) {
    if (lane < nprod) {
      for (int j = lane; j < pages_per_cta; j += nprod) {
        int st = j % S;
        if (j >= S) mbar_wait(&empty[st], ((j / S) - 1) & 1);
        stv(&tag[st], j);
        size_t off = ((page0 + j) * heads + head) * 4096;
        mbar_expect(&full[st], 8192);
        bulk(smem + st * 8192, kp + off, 4096, &full[st]);
        bulk(smem + st * 8192 + 4096, vp + off, 4096, &full[st]);
      }
    }
    return;
  }
  float acc = 0.f;
  for (int j = warp; j < pages_per_cta; j += ncons) {
    int st = j % S;
    while (ldv(&tag[st]) != j) {}
    mbar_wait(&full[st], (j / S) & 1);
    acc += (float)smem[st * 8192 + lane * 4];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  if (acc == 1234.5f) sink[0] = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int heads = 8;
  size_t plane = (size_t)2 << 30;
  uint8_t *kp, *vp; cudaMalloc(&kp, plane); cudaMalloc(&vp, plane); cudaMemset(kp, 1, plane); cudaMemset(vp, 1, plane);
  float* sink; cudaMalloc(&sink, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  size_t smem = S * 8192 + 2 * S * 8 + S * 4;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  size_t total_pages = plane / (heads * 4096);
  int grid = sms;  // groups of `heads` CTAs share a page range
  int pages_per_cta = (int)(total_pages / ((grid + heads - 1) / heads)) ;
  int cfg[][2] = {{1, 1}, {1, 6}, {5, 1}, {5, 6}, {15, 6}, {15, 1}, {3, 6}};
  for (auto& c : cfg) {
    k<<<grid, (c[1] + 1) * 32, smem>>>(kp, vp, pages_per_cta, c[0], c[1], heads, sink);
    cudaEventRecord(e0);
    k<<<grid, (c[1] + 1) * 32, smem>>>(kp, vp, pages_per_cta, c[0], c[1], heads, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("nprod=%2d ncons=%d : %7.1f GB/s (%s)\n", c[0], c[1], (double)grid * pages_per_cta * 8192 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
}
