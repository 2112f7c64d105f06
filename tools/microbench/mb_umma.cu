// Microbenchmark: issue + completion cost of the decode kernel's tcgen05.mma shapes on B200.
//   QK: SS, M=128, N in {16,64,128,256}, K=16, K-major SW128 A and B
//   PV: TS, M=128, N=128, K=16, A from TMEM, B MN-major SW128
// One thread issues R back-to-back MMAs into one accumulator, commits, waits; cycles / MMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_common.cuh"

using namespace mv;

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void mma_ss_e(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_ts_e(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}

__global__ void __launch_bounds__(128, 1) umma_bench(int mode, int N, int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) ((uint4*)smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  tc::fence_proxy_async();
  if (mode >= 3 && mode < 6 && threadIdx.x < 32) {
    // whole warp runs the loop (uniform descriptors), one elected lane issues
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint32_t idqk = tc::idesc_bf16(128, N, 0, 0), idpv = tc::idesc_bf16(128, 128, 0, 1);
    const uint64_t da = tc::sw128_desc(a, 16, 1024), db = tc::sw128_desc(b, 16, 1024), dv = tc::sw128_desc(b, 2048, 1024);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (mode == 3) {
        const int k = r & 7;
        const uint32_t oq = ((k >> 2) * 16384 + (k & 3) * 32) >> 4;
        mma_ss_e(tmem, da + oq, db + oq, idqk, r > 0);
      } else if (mode == 4) {
        const int p = r & 3;
        mma_ts_e(tmem + 128, tmem + p * 8, dv + ((p * 4096) >> 4), idpv, r > 0);
      } else {
        const int k = r % 12;
        if (k < 8) {
          const uint32_t oq = ((k >> 2) * 16384 + (k & 3) * 32) >> 4;
          mma_ss_e(tmem, da + oq, db + oq, idqk, k > 0);
        } else {
          mma_ts_e(tmem + 256, tmem + (k - 8) * 8, dv + (((k - 8) * 4096) >> 4), idpv, 1);
        }
      }
    }
    long long t1 = clock64();
    if (elect_one()) tc::mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  if (mode >= 6 && threadIdx.x < 32 && (mode == 7 || threadIdx.x == 0)) {
    // unrolled groups of 8 k-steps, descriptors = base + compile-time offsets
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint32_t idqk = tc::idesc_bf16(128, N, 0, 0);
    const uint64_t da = tc::sw128_desc(a, 16, 1024), db = tc::sw128_desc(b, 16, 1024);
    long long t0 = clock64();
    for (int r = 0; r < reps; r += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t oq = ((k >> 2) * 16384 + (k & 3) * 32) >> 4;
        if (mode == 7) mma_ss_e(tmem, da + oq, db + oq, idqk, k > 0);
        else tc::mma_ss(tmem, da + oq, db + oq, idqk, k > 0);
      }
    }
    long long t1 = clock64();
    if (mode == 6 || elect_one()) tc::mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  if (mode < 3 && threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint32_t idqk = tc::idesc_bf16(128, N, 0, 0), idpv = tc::idesc_bf16(128, 128, 0, 1);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (mode == 0) {
        const int k = r & 7;
        const uint32_t oq = (k >> 2) * 16384 + (k & 3) * 32, ok = (k >> 2) * 16384 + (k & 3) * 32;
        tc::mma_ss(tmem, tc::sw128_desc(a + oq, 16, 1024), tc::sw128_desc(b + ok, 16, 1024), idqk, r > 0);
      } else if (mode == 1) {
        const int p = r & 3;
        tc::mma_ts(tmem + 128, tmem + p * 8, tc::sw128_desc(b + p * 4096, 2048, 1024), idpv, r > 0);
      } else {
        // decode block: 8 QK (N) then 4 PV
        const int k = r % 12;
        if (k < 8) {
          const uint32_t oq = (k >> 2) * 16384 + (k & 3) * 32, ok = (k >> 2) * 16384 + (k & 3) * 32;
          tc::mma_ss(tmem, tc::sw128_desc(a + oq, 16, 1024), tc::sw128_desc(b + ok, 16, 1024), idqk, k > 0);
        } else {
          tc::mma_ts(tmem + 256, tmem + (k - 8) * 8, tc::sw128_desc(b + (k - 8) * 4096, 2048, 1024), idpv, 1);
        }
      }
    }
    long long t1 = clock64();
    tc::mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  __syncthreads();
  if (threadIdx.x < 32) { tc::fence_after(); tc::tmem_dealloc(tmem, 512); }
}

extern __shared__ __align__(1024) uint8_t smem_sym[];
// mode 10: NW warps issue concurrently (lane 0 each, unrolled), each into its own D columns
__global__ void __launch_bounds__(128, 1) umma_bench3(int nw, int N, int reps, unsigned long long* out) {
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) ((uint4*)smem_sym)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { for (int w = 0; w < 4; ++w) mbar_init(&bar[w], 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  tc::fence_proxy_async();
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && w < nw) {
    const uint32_t a = smem_u32(smem_sym), b = a + 32768;
    const uint32_t idqk = tc::idesc_bf16(128, N, 0, 0);
    const uint64_t da = tc::sw128_desc(a, 16, 1024), db = tc::sw128_desc(b, 16, 1024);
    long long t0 = clock64();
    for (int r = 0; r < reps; r += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t oq = ((k >> 2) * 16384 + (k & 3) * 32) >> 4;
        tc::mma_ss(tmem + w * 128, da + oq, db + oq, idqk, k > 0);
      }
    }
    long long t1 = clock64();
    tc::mma_commit(&bar[w]);
    mbar_wait(&bar[w], 0);
    long long t2 = clock64();
    if (blockIdx.x == 0 && w == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  __syncthreads();
  if (threadIdx.x < 32) { tc::fence_after(); tc::tmem_dealloc(tmem, 512); }
}
// mode 8: warp-converged loop, descriptors from the smem symbol, C++ elect branch around one asm
// mode 9: same, elect predicate inside the asm
__global__ void __launch_bounds__(128, 1) umma_bench2(int mode, int N, int reps, unsigned long long* out) {
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) ((uint4*)smem_sym)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, tslot, 0);
  tc::fence_proxy_async();
  if (threadIdx.x < 32) {
    const uint32_t a = smem_u32(smem_sym), b = a + 32768;
    const uint32_t idqk = tc::idesc_bf16(128, 64, 0, 0);
    const uint64_t da = tc::sw128_desc(a, 16, 1024), db = tc::sw128_desc(b, 16, 1024);
    long long t0 = clock64();
    for (int r = 0; r < reps; r += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t oq = ((k >> 2) * 16384 + (k & 3) * 32) >> 4;
        if (mode == 8) {
          if (elect_one()) tc::mma_ss(tmem, da + oq, db + oq, idqk, k > 0);
          __syncwarp();
        } else {
          mma_ss_e(tmem, da + oq, db + oq, idqk, k > 0);
        }
      }
    }
    long long t1 = clock64();
    if (elect_one()) tc::mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  __syncthreads();
  if (threadIdx.x < 32) { tc::fence_after(); tc::tmem_dealloc(tmem, 512); }
}

// mode 11: the decode block sequence, unrolled: 8 QK (TS, A = Q in TMEM, N = 64) + 4 PV (TS, N = 128,
// MN-major V) + commit; mode 12: same with QK SS (A = Q in smem)
__global__ void __launch_bounds__(128, 1) umma_block(int mode, int reps, unsigned long long* out) {
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) ((uint4*)smem_sym)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  tc::fence_proxy_async();
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem_sym), b = a + 32768;
    const uint32_t idqk = tc::idesc_bf16(128, 64, 0, 0), idpv = tc::idesc_bf16(128, 128, 0, 1);
    const uint64_t qd = tc::sw128_desc(a, 16, 1024), kd = tc::sw128_desc(b, 16, 1024);
    const uint64_t vd = tc::sw128_desc(b + 16384, 2048, 1024);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t scol = tmem + (r & 1) * 64, ocol = tmem + 128 + (r & 1) * 128;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (mode >= 13) break;
        const uint64_t ko = kd + (uint64_t)(((k >> 2) * 8192 + (k & 3) * 32) >> 4);
        if (mode == 11) tc::mma_ts(scol, tmem + 384 + k * 8, ko, idqk, k > 0);
        else tc::mma_ss(scol, qd + (uint64_t)(((k >> 2) * 16384 + (k & 3) * 32) >> 4), ko, idqk, k > 0);
      }
      if (mode >= 24) {
        // 8 QK-like SS N=64, then 4 more SS MMAs into another D with: 24 same idesc, 25 N=128 K-major,
        // 26 N=128 MN-major B, 27 N=64 MN-major B
        const uint32_t id2 = mode == 24 ? idqk : mode == 25 ? tc::idesc_bf16(128, 128, 0, 0)
                             : mode == 27 ? tc::idesc_bf16(128, 64, 0, 1) : tc::idesc_bf16(128, 128, 0, 1);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          tc::mma_ss(scol, qd + (uint64_t)((((k & 7) >> 2) * 16384 + (k & 3) * 32) >> 4),
                     kd + (uint64_t)((((k & 7) >> 2) * 8192 + (k & 3) * 32) >> 4), idqk, k > 0);
        if (mode == 29 || mode == 31) tc::mma_commit(&bar[1]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (mode >= 30) tc::mma_ts(ocol, tmem + 384 + k * 8, vd + (uint64_t)((k * 4096) >> 4), id2, 1);
          else tc::mma_ss(ocol, qd + (uint64_t)(((k & 3) * 32) >> 4), vd + (uint64_t)((k * 4096) >> 4), id2, 1);
        }
        if (mode >= 28) tc::mma_commit(&bar[1]);
        continue;
      }
      if (mode == 21 || mode == 22 || mode == 23) {
        // 12 SS N=64 MMAs; 21: D alternates per iteration; 22: fixed D; 23: D alternates every 4 MMAs
#pragma unroll
        for (int k = 0; k < 12; ++k) {
          const uint32_t dd = mode == 22 ? tmem : (mode == 21 ? scol : tmem + ((k >> 2) & 1) * 64);
          tc::mma_ss(dd, qd + (uint64_t)((((k & 7) >> 2) * 16384 + (k & 3) * 32) >> 4),
                     kd + (uint64_t)((((k & 7) >> 2) * 8192 + (k & 3) * 32) >> 4), idqk, 1);
        }
        continue;
      }
      if (mode >= 18) {
        const uint64_t pd = tc::sw128_desc(a + 65536 - 32768 + 0, 16, 1024);  // P tile in smem (K-major)
        const int nqk = mode == 20 ? 2 : 1;
        for (int x = 0; x < nqk; ++x) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint64_t ko = kd + (uint64_t)(((k >> 2) * 8192 + (k & 3) * 32) >> 4);
            if (mode == 18) tc::mma_ts(tmem + x * 64, tmem + 384 + k * 8, ko, idqk, k > 0);
            else tc::mma_ss(tmem + x * 64, qd + (uint64_t)(((k >> 2) * 16384 + (k & 3) * 32) >> 4), ko, idqk, k > 0);
          }
        }
        for (int x = 0; x < nqk; ++x) {
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            if (mode == 20) tc::mma_ts(ocol, tmem + x * 64 + p * 8, vd + (uint64_t)((p * 4096) >> 4), idpv, 1);
            else tc::mma_ss(ocol, pd + (uint64_t)((p * 32) >> 4), vd + (uint64_t)((p * 4096) >> 4), idpv, 1);
          }
        }
        tc::mma_commit(&bar[1]);
        if (mode == 20) ++r;
        continue;
      }
      if (mode >= 13 && mode <= 15) {  // PV-only variants
        const uint32_t pc = tmem + ((r + 1) & 1) * 64;
        const uint32_t id = mode == 13 ? idpv : (mode == 14 ? tc::idesc_bf16(128, 128, 0, 0) : tc::idesc_bf16(128, 64, 0, 1));
#pragma unroll
        for (int p = 0; p < 8; ++p) tc::mma_ts(ocol, pc + (p & 3) * 8, vd + (uint64_t)(((p & 3) * 4096) >> 4), id, 1);
        tc::mma_commit(&bar[1]);
        continue;
      }
      if (mode == 11 || mode == 12) tc::mma_commit(&bar[1]);
      const uint32_t pc = tmem + ((r + 1) & 1) * 64;
      tc::mma_ts(ocol, pc, vd, idpv, 1);
      tc::mma_ts(ocol, pc + 8, vd + (4096 >> 4), idpv, 1);
      tc::mma_ts(ocol, pc + 16, vd + (8192 >> 4), idpv, 1);
      tc::mma_ts(ocol, pc + 24, vd + (12288 >> 4), idpv, 1);
      if (mode != 17) tc::mma_commit(&bar[1]);
    }
    long long t1 = clock64();
    tc::mma_commit(&bar[0]);
    mbar_wait(&bar[0], 0);
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  __syncthreads();
  if (threadIdx.x < 32) { tc::fence_after(); tc::tmem_dealloc(tmem, 512); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  cudaFuncSetAttribute(umma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const char* names[8] = {"QK SS M128 K16", "PV TS M128 N128 K16", "block 8xQK + 4xPV", "warp QK SS", "warp PV TS", "warp block", "thread QK unrolled", "warp QK unrolled"};
  for (int grid : {1, 148})
    for (int mode = 0; mode < 8; ++mode)
      for (int N : {16, 64, 128, 256}) {
        if ((mode == 1 || mode == 4) && N != 128) continue;
        if (grid > 1 && N != 64) continue;
        const int reps = 1200;
        umma_bench<<<grid, 128, 100 * 1024>>>(mode, N, reps, d);
        umma_bench<<<grid, 128, 100 * 1024>>>(mode, N, reps, d);
        unsigned long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("grid %3d %-22s N=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma (%s)\n", grid, names[mode], N,
               (double)h[0] / reps, (double)h[1] / reps, cudaGetErrorString(cudaGetLastError()));
        fflush(stdout);
      }
  cudaFuncSetAttribute(umma_bench2, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int mode = 8; mode < 10; ++mode) {
    const int reps = 1200;
    umma_bench2<<<1, 128, 100 * 1024>>>(mode, 64, reps, d);
    umma_bench2<<<1, 128, 100 * 1024>>>(mode, 64, reps, d);
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("mode %d N=64: issue %.1f cyc/mma, complete %.1f (%s)\n", mode, (double)h[0] / reps, (double)h[1] / reps,
           cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
  }
  cudaFuncSetAttribute(umma_bench3, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int nw = 1; nw <= 4; nw *= 2)
    for (int N : {64, 128}) {
      const int reps = 1200;
      umma_bench3<<<1, 128, 100 * 1024>>>(nw, N, reps, d);
      umma_bench3<<<1, 128, 100 * 1024>>>(nw, N, reps, d);
      unsigned long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("%d issuing warps N=%d: per-warp %.1f cyc/mma, aggregate %.1f cyc/mma (%s)\n", nw, N,
             (double)h[1] / reps, (double)h[1] / reps / nw, cudaGetErrorString(cudaGetLastError()));
      fflush(stdout);
    }
  cudaFuncSetAttribute(umma_block, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int mode = 11; mode <= 31; ++mode) {
    if (mode < 24) continue;
    if (mode == 16 || mode == 17) continue;
    const int reps = 200;
    umma_block<<<148, 128, 100 * 1024>>>(mode, reps, d);
    umma_block<<<148, 128, 100 * 1024>>>(mode, reps, d);
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("decode block mode %d (%s): issue %.0f cyc/block, complete %.0f cyc/block (%s)\n", mode,
           mode == 11 ? "QK TS" : mode == 12 ? "QK SS" : mode == 13 ? "8 PV MN-major" : mode == 14 ? "8 PV K-major B" : mode == 15 ? "8 PV N=64" : mode == 16 ? "block, 1 commit" : mode == 17 ? "block, no commit" : mode == 18 ? "QK TS + PV SS" : mode == 19 ? "QK SS + PV SS" : mode == 20 ? "2x QK SS + 2x PV TS" : mode == 21 ? "12 MMA, D flips per iter" : mode == 22 ? "12 MMA, fixed D" : mode == 23 ? "12 MMA, D flips every 4" : mode == 24 ? "8+4 same idesc" : mode == 25 ? "8+4 N128 Kmaj" : mode == 26 ? "8+4 N128 MNmaj" : mode == 27 ? "8+4 N64 MNmaj" : mode == 28 ? "8+4, 1 commit" : mode == 29 ? "8+4, 2 commits" : mode == 30 ? "8+4 PV TS, 1 commit" : "8+4 PV TS, 2 commits", (double)h[0] / reps, (double)h[1] / reps, cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
  }
  return 0;
}
