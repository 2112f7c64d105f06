// Microbenchmark: issue cost of 1-D bulk copies (UBLKCP) and L2 prefetches from one thread vs all
// lanes of a warp (one copy per lane per instruction).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"

using namespace mv;
extern __shared__ __align__(1024) uint8_t smem_b[];

__global__ void bulk_issue(const uint8_t* src, int mode, int reps, unsigned long long* out) {
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  const int lane = threadIdx.x;
  const uint8_t* base = src + (size_t)blockIdx.x * (1 << 22);
  long long t0 = clock64();
  uint32_t total = 0;
  for (int r = 0; r < reps; ++r) {
    // one round = 32 copies of 2 KiB into smem (64 KiB)
    if (mode == 0) {
      if (lane == 0) {
        mbar_arrive_expect_tx(&bar, 32 * 2048);
        for (int c = 0; c < 32; ++c) bulk_g2s(smem_b + c * 2048, base + ((r * 32 + c) % 2048) * 2048, 2048, &bar);
      }
    } else if (mode == 1) {
      if (lane == 0) mbar_arrive_expect_tx(&bar, 32 * 2048);
      __syncwarp();
      bulk_g2s(smem_b + lane * 2048, base + ((r * 32 + lane) % 2048) * 2048, 2048, &bar);
    } else if (mode == 2) {
      if (lane == 0) for (int c = 0; c < 32; ++c) prefetch_l2(base + ((r * 32 + c) % 2048) * 2048, 2048);
    } else {
      prefetch_l2(base + ((r * 32 + lane) % 2048) * 2048, 2048);
    }
    if (mode <= 1) {
      mbar_wait(&bar, r & 1);
    }
    total += 32;
  }
  long long t1 = clock64();
  if (blockIdx.x == 0 && lane == 0) { out[0] = t1 - t0; out[1] = total; }
}

int main() {
  uint8_t* src; cudaMalloc(&src, (size_t)148 << 22);
  cudaMemset(src, 1, (size_t)148 << 22);
  unsigned long long* d; cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bulk_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  const char* names[4] = {"copies, lane 0 loop", "copies, 32 lanes", "prefetch, lane 0 loop", "prefetch, 32 lanes"};
  for (int grid : {1, 148})
    for (int mode = 0; mode < 4; ++mode) {
      bulk_issue<<<grid, 32, 80 * 1024>>>(src, mode, 50, d);
      bulk_issue<<<grid, 32, 80 * 1024>>>(src, mode, 50, d);
      unsigned long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("grid %3d %-24s: %.1f cyc per copy (incl. completion for copies) (%s)\n", grid, names[mode],
             (double)h[0] / h[1], cudaGetErrorString(cudaGetLastError()));
      fflush(stdout);
    }
  return 0;
}
