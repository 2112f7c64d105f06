// The prefill kernel's tensor-core sequence per 128 x 128 tile in isolation (one CTA, one SM):
//   QK: 8 x SS M128 N128 K16 (Q, K K-major SW128 in smem) into S buffer b, commit
//   PV: 8 x TS M128 N128 K16 (P from TMEM, V MN-major SW128 in smem) into O, commit
// Cycles per tile for: one issuing thread (QK then PV), two issuing warps (QK / PV), QK only,
// PV only, and QK with N = 256 (two k tiles per MMA, half the instructions).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../include -I../../paper_2506_09991_b200/csrc
//        -o mb_pf_mma mb_pf_mma.cu
#include <cstdio>

#include "tc_common.cuh"

namespace mv {
void set_error(const std::string&) {}
mv_status fail(mv_status st, const std::string&) { return st; }
}  // namespace mv
using namespace mv;

constexpr int kHalf = 128 * 128;  // SW128 half tile: 128 rows x 64 dims bf16
constexpr uint32_t kIdQK = tc::idesc_bf16(128, 128, 0, 0), kIdQK256 = tc::idesc_bf16(128, 256, 0, 0);
constexpr uint32_t kIdPV = tc::idesc_bf16(128, 128, 0, 1);

template <int B>
__device__ __forceinline__ void qk(uint32_t tm, uint64_t qd, uint64_t kd) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint64_t off = (uint64_t)(((k >> 2) * kHalf + (k & 3) * 32) >> 4);
    tc::mma_ss(tm + B * 128, qd + off, kd + off, kIdQK, k > 0 ? 1u : 0u);
  }
}
__device__ __forceinline__ void qk256(uint32_t tm, uint64_t qd, uint64_t kd) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint64_t off = (uint64_t)(((k >> 2) * kHalf + (k & 3) * 32) >> 4);
    const uint64_t koff = (uint64_t)(((k >> 2) * 2 * kHalf + (k & 3) * 32) >> 4);
    tc::mma_ss(tm, qd + off, kd + koff, kIdQK256, k > 0 ? 1u : 0u);
  }
}
template <int B>
__device__ __forceinline__ void pv(uint32_t tm, uint64_t vd) {
#pragma unroll
  for (int k = 0; k < 8; ++k)
    tc::mma_ts(tm + 384, tm + B * 128 + k * 8, vd + (uint64_t)((k * 2048) >> 4), kIdPV, 1u);
}

// MODE 0: one thread QK+PV; 1: two warps (QK warp 0, PV warp 1); 2: QK only; 3: PV only; 4: QK N=256
// (per 2 tiles) + 2 x PV, one thread.  LOAD bit 0: 8 warps (2..9) stream TMEM ld x64 / st x32 per row
// like the softmax; bit 1: warp 10 streams 16 KiB bulk copies global -> smem (the TMA K/V traffic).
__device__ __forceinline__ void mb_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ volatile int g_stop;
template <int MODE, int LOAD = 0>
__global__ void __launch_bounds__(352, 1) bench(int reps, long long* out, const uint8_t* gsrc, long long* side) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar[2];
  __shared__ uint64_t cbar[2];
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&cbar[0], 1);
    mbar_init(&cbar[1], 1);
    stop = 0;
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc(&slot, 512);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = slot;
  const uint64_t qd = tc::sw128_desc(smem_u32(smem), 16, 1024);
  const uint64_t kd = tc::sw128_desc(smem_u32(smem + 32768), 16, 1024);
  const uint64_t vd = tc::sw128_desc(smem_u32(smem + 98304), kHalf, 1024);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  long long t0 = clock64();
  if (w >= 2 && w < 10) {
    long long n = 0;
    if (LOAD & 1) {
      const uint32_t base = tm + ((uint32_t)((w & 3) * 32) << 16) + ((w - 2) >> 2) * 64;
      float v[32];
      while (!stop) {
        tc::tmem_ld32(base, v);
        tc::tmem_ld32(base + 32, v);
        tc::tmem_wait_ld();
        uint32_t u[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) u[k] = __float_as_uint(v[2 * k] + v[2 * k + 1]);
        tc::tmem_stNu<16>(base + 256, u);
        tc::tmem_wait_st();
        ++n;
      }
    }
    if (lane == 0) side[w] = n;
    return;
  }
  if (w == 10) {
    long long n = 0;
    if ((LOAD & 2) && lane == 0) {
      uint32_t ph[2] = {0, 0};
      for (long long i = 0; !stop; ++i) {
        const int b = i & 1;
        if (i >= 2) { mbar_wait(&cbar[b], ph[b]); ph[b] ^= 1; }
        mbar_arrive_expect_tx(&cbar[b], 16384);
        mb_bulk_g2s(smem + 131072 + b * 16384, gsrc + ((i * 16384) & ((64 << 20) - 1)), 16384, &cbar[b]);
        ++n;
      }
      mbar_wait(&cbar[0], ph[0]);
      mbar_wait(&cbar[1], ph[1]);
    }
    if (lane == 0) side[10] = n;
    return;
  }
  if ((threadIdx.x & 31) == 0) {
    if (MODE == 0 && w == 0) {
      for (int r = 0; r < reps; ++r) {
        if (r & 1) { qk<1>(tm, qd, kd); pv<0>(tm, vd); }
        else { qk<0>(tm, qd, kd); pv<1>(tm, vd); }
        tc::mma_commit(&bar[0]);
      }
    } else if (MODE == 1) {
      for (int r = 0; r < reps; ++r) {
        if (w == 0) { if (r & 1) qk<1>(tm, qd, kd); else qk<0>(tm, qd, kd); }
        else { if (r & 1) pv<0>(tm, vd); else pv<1>(tm, vd); }
        tc::mma_commit(&bar[w]);
      }
    } else if (MODE == 2 && w == 0) {
      for (int r = 0; r < reps; ++r) { if (r & 1) qk<1>(tm, qd, kd); else qk<0>(tm, qd, kd); tc::mma_commit(&bar[0]); }
    } else if (MODE == 3 && w == 0) {
      for (int r = 0; r < reps; ++r) { if (r & 1) pv<0>(tm, vd); else pv<1>(tm, vd); tc::mma_commit(&bar[0]); }
    } else if (MODE == 4 && w == 0) {
      for (int r = 0; r < reps; r += 2) {
        qk256(tm, qd, kd);
        pv<0>(tm, vd);
        pv<1>(tm, vd);
        tc::mma_commit(&bar[0]);
      }
    }
  }
  __syncwarp();
  // drain: a final commit per issuing thread, then wait
  if ((threadIdx.x & 31) == 0 && (w == 0 || MODE == 1)) {
    tc::mma_commit(&bar[w]);
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0 && (w == 0 || MODE == 1)) {
    const int commits = (MODE == 4 ? reps / 2 : reps) + 1;
    mbar_wait(&bar[w], (commits - 1) & 1);
  }
  asm volatile("bar.sync 1, 64;");
  long long t2 = clock64();
  if (threadIdx.x == 0) stop = 1;
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc::fence_after(); tc::tmem_dealloc(tm, 512); }
}

template <int MODE, int LOAD = 0>
void run(const char* name) {
  long long *d, *side;
  uint8_t* src;
  cudaMalloc(&d, 16);
  cudaMalloc(&side, 16 * 8);
  cudaMalloc(&src, 64 << 20);
  cudaMemset(side, 0, 128);
  cudaFuncSetAttribute(bench<MODE, LOAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 166 * 1024);
  const int reps = 400;
  bench<MODE, LOAD><<<1, 352, 166 * 1024>>>(reps, d, src, side);
  bench<MODE, LOAD><<<1, 352, 166 * 1024>>>(reps, d, src, side);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2], hs[16];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(hs, side, 128, cudaMemcpyDeviceToHost);
  printf("%-44s complete %6.0f cyc per tile (floor 1024)  softmax-like steps/warp %lld  bulk 16K copies %lld (%.0f B/cyc)  %s\n",
         name, (double)h[1] / reps, hs[2], hs[10], hs[10] * 16384.0 / h[1], cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(side);
  cudaFree(src);
}

int main() {
  run<2>("QK only (8 SS N128)");
  run<3>("PV only (8 TS N128)");
  run<0>("QK + PV, one thread");
  run<1>("QK warp + PV warp");
  run<4>("QK N256 per 2 tiles + PV, one thread");
  run<0, 1>("QK+PV + TMEM ld/st traffic");
  run<0, 2>("QK+PV + bulk copies");
  run<0, 3>("QK+PV + TMEM traffic + bulk copies");
  run<4, 3>("QK N256 + PV + TMEM + bulk");
  run<1, 3>("QK warp + PV warp + TMEM + bulk");
  return 0;
}
