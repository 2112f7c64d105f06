// Microbenchmark: achievable HBM bandwidth of the decode kernel's access pattern — 1-D bulk
// copies (cp.async.bulk) of randomly placed page-head blocks into a shared-memory ring, one
// persistent CTA per SM, two issuing lanes (as decode_tc's TMA warp), consumer releasing slots
// immediately.  Sweeps the block size and the ring depth.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2506_09991_b200/csrc -o mb_gather mb_gather.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "common.cuh"

using namespace mv;
extern __shared__ __align__(1024) uint8_t smem_g[];

constexpr int kMaxSlots = 12;

__global__ void __launch_bounds__(64, 1) gather(const uint8_t* pool, const uint32_t* pages, int n_per_cta,
                                                int page_bytes, int pages_per_slot, int slots, int issuers,
                                                unsigned long long* bytes_out) {
  __shared__ uint64_t full[kMaxSlots], empty[kMaxSlots];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < slots; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t* my = pages + (size_t)blockIdx.x * n_per_cta;
  const int n_blocks = n_per_cta / pages_per_slot;
  const int slot_bytes = page_bytes * pages_per_slot;
  if (warp == 0 && lane < issuers) {  // producer: `issuers` lanes split each slot's pages
    for (int b = 0; b < n_blocks; ++b) {
      const int s = b % slots;
      if (b >= slots) mbar_wait(&empty[s], ((b / slots) - 1) & 1);
      if (lane == 0) mbar_arrive_expect_tx(&full[s], slot_bytes);
      for (int p = lane; p < pages_per_slot; p += issuers)
        bulk_g2s(smem_g + s * slot_bytes + p * page_bytes, pool + (size_t)my[b * pages_per_slot + p] * page_bytes,
                 page_bytes, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {  // consumer
    for (int b = 0; b < n_blocks; ++b) {
      const int s = b % slots;
      mbar_wait(&full[s], (b / slots) & 1);
      mbar_arrive(&empty[s]);
    }
    atomicAdd(bytes_out, (unsigned long long)n_blocks * slot_bytes);
  }
}

int main() {
  const size_t pool_bytes = 4ull << 30;  // 4 GB pool (>> L2)
  uint8_t* pool;
  cudaMalloc(&pool, pool_bytes);
  cudaMemset(pool, 1, pool_bytes);
  int sms = 148;
  unsigned long long* d_bytes;
  cudaMalloc(&d_bytes, 8);
  for (int page_bytes : {4096}) {
    const size_t n_pages_pool = pool_bytes / page_bytes;
    const int per_cta = (int)((1ull << 30) / page_bytes / sms);  // 1 GB moved in total
    std::vector<uint32_t> h((size_t)per_cta * sms);
    uint64_t x = 88172645463325252ull;
    for (auto& v : h) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; v = (uint32_t)(x % n_pages_pool); }
    uint32_t* d_pages;
    cudaMalloc(&d_pages, h.size() * 4);
    cudaMemcpy(d_pages, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    for (int slot_kb : {16}) {
      const int pps = std::max(1, slot_kb * 1024 / page_bytes);
      for (int issuers : {4})
      for (int slots : {6, 9, 11, 12}) {
        if (issuers > pps) continue;
        const int smem = slots * pps * page_bytes;
        if (smem > 220 * 1024) continue;
        cudaFuncSetAttribute(gather, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        gather<<<sms, 64, smem>>>(pool, d_pages, per_cta, page_bytes, pps, slots, issuers, d_bytes);  // warm
        cudaMemset(d_bytes, 0, 8);
        cudaEventRecord(e0);
        gather<<<sms, 64, smem>>>(pool, d_pages, per_cta, page_bytes, pps, slots, issuers, d_bytes);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long b;
        cudaMemcpy(&b, d_bytes, 8, cudaMemcpyDeviceToHost);
        printf("page %6d B, slot %2d KB, %d issuing lanes, %2d slots (%3d KB/SM): %7.1f GB/s (%s)\n", page_bytes,
               pps * page_bytes / 1024, issuers, slots, smem / 1024, b / (ms * 1e6),
               cudaGetErrorString(cudaGetLastError()));
      }
    }
    cudaFree(d_pages);
  }
  return 0;
}
