// The prefill softmax step in isolation (one CTA, no tensor core): each warp loads its 64 score
// columns of a 128-row tile from TMEM, exponentiates (FFMA2 scale, MUFU.EX2 + 1 pair in 8 on the
// FMA pipe, FADD2 sums, bf16 pack), OR-reduces the sum guard over the column-half pair and stores P.
// Cycles per step per warp, by variant, at 2 or 4 warps per SMSP.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../include -I../../paper_2506_09991_b200/csrc
//        -o mb_softmax mb_softmax.cu
#include <cstdio>

#include "tc_common.cuh"

namespace mv {
void set_error(const std::string&) {}
mv_status fail(mv_status st, const std::string&) { return st; }
}  // namespace mv
using namespace mv;

constexpr int kIters = 512;

__device__ __forceinline__ bool pair_any(int id, int cnt, bool pred) {
  uint32_t out;
  asm volatile(
      "{\n.reg .pred pi, po;\nsetp.ne.u32 pi, %1, 0;\nbarrier.cta.red.or.pred po, %2, %3, pi;\nselp.u32 %0, 1, 0, po;\n}\n"
      : "=r"(out)
      : "r"((uint32_t)pred), "r"(id), "r"(cnt)
      : "memory");
  return out != 0;
}

// MODE bit 0: pair barrier; bit 1: TMEM ld / st; bit 2: poly pairs (1 in 8)
// MODE bit 3: one extra warp keeps the tensor core busy meanwhile (S-like SS MMAs into columns
// 256-383, P.V-like TS MMAs reading A from columns 192-255 into 384-511), as the prefill kernel's MMA warp does
template <int MODE>
__global__ void __launch_bounds__(512, 1) bench(float* out, long long* cyc, float scale) {
  __shared__ uint32_t slot;
  __shared__ volatile int done_flag;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ __align__(8) uint64_t mbar2;
  extern __shared__ __align__(1024) uint8_t dsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  if (threadIdx.x == 0) {
    done_flag = 0;
    mbar_init(&mbar, 1);
    mbar_init(&mbar2, 1);
    fence_mbar_init();
  }
  if (MODE & 8) {
    for (int i = threadIdx.x; i < 2 * 32768 / 16; i += blockDim.x) reinterpret_cast<uint4*>(dsm)[i] = make_uint4(0, 0, 0, 0);
    tc::fence_proxy_async();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if ((MODE & 512) && warp == nw - 1) return;  // extra warp idle: launch shape only
  if ((MODE & 8) && !(MODE & 512) && warp == nw - 1) {
    long long issued = 0;
    if (lane == 0) {
      uint8_t* al = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
      const uint64_t ad = tc::sw128_desc(smem_u32(al), 16, 1024), bd = tc::sw128_desc(smem_u32(al + 32768), 16, 1024);
      const uint32_t id = tc::idesc_bf16(128, 128, 0, 0), idv = tc::idesc_bf16(128, 128, 0, 1);
      uint32_t ph = 0, ph2 = 0;
      const long long tm0 = clock64();
      for (int b = 0; b < 200000 && !done_flag; ++b) {
        if (MODE & 2048) {  // pipelined: two batches in flight, throughput-bound
          uint64_t* mb = (b & 1) ? &mbar2 : &mbar;
          if (b >= 2) {
            if (b & 1) { mbar_wait(&mbar2, ph2); ph2 ^= 1; }
            else { mbar_wait(&mbar, ph); ph ^= 1; }
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) tc::mma_ss(slot + 256, ad + (k * 2), bd + (k * 2), id, k > 0);
#pragma unroll
          for (int k = 0; k < 8; ++k) tc::mma_ts(slot + 384, slot + 192 + k * 8, bd + (k * 128), idv, 1);
          tc::mma_commit(mb);
          issued += 16;
          continue;
        }
        if (MODE & 128) {  // spin on a barrier that does not complete for ~the MMA batch time
          const long long t = clock64();
          while (clock64() - t < 1024 && !mbar_test(&mbar, ph)) {
          }
          continue;
        }
        if (MODE & 256) {  // MMAs, then sleep-poll instead of spinning
#pragma unroll
          for (int k = 0; k < 8; ++k) tc::mma_ss(slot + 256, ad + (k * 2), bd + (k * 2), id, k > 0);
#pragma unroll
          for (int k = 0; k < 8; ++k) tc::mma_ts(slot + 384, slot + 192 + k * 8, bd + (k * 128), idv, 1);
          tc::mma_commit(&mbar);
          while (!mbar_test(&mbar, ph)) __nanosleep(200);
          ph ^= 1;
          issued += 16;
          continue;
        }
        if (!(MODE & 64)) {
#pragma unroll
          for (int k = 0; k < 8; ++k) tc::mma_ss(slot + 256, ad + (k * 2), bd + (k * 2), id, k > 0);
        }
        if (!(MODE & 32)) {
#pragma unroll
          for (int k = 0; k < 8; ++k) tc::mma_ts(slot + 384, slot + 192 + k * 8, bd + (k * 128), idv, 1);
        }
        tc::mma_commit(&mbar);
        mbar_wait(&mbar, ph);
        ph ^= 1;
        issued += (MODE & 96) ? 8 : 16;
      }
      if (MODE & 2048) {
        mbar_wait(&mbar, ph);
        mbar_wait(&mbar2, ph2);
      }
      cyc[30] = clock64() - tm0;
    }
    __syncwarp();
    if (lane == 0) cyc[31] = issued;
    tc::fence_before();
    __syncthreads();  // final
    return;
  }
  const int quarter = warp & 3, c = (warp >> 2) & 1, grp = warp >> 3;  // grp: second pair on the SMSP
  const uint32_t base = slot + ((uint32_t)(quarter * 32) << 16) + grp * 256;
  {
    float init[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) init[k] = (lane * 7 + k * 13 % 29) * 0.01f - 1.f;
    tc::tmem_st32(base + c * 64, init);
    tc::tmem_st32(base + c * 64 + 32, init);
    tc::tmem_wait_st();
  }
  asm volatile("bar.sync 14, %0;" ::"r"((MODE & 8) ? (nw - 1) * 32 : nw * 32));
  float v[64];
#pragma unroll
  for (int k = 0; k < 64; ++k) v[k] = (lane + k) * 0.01f;

  float l = 0.f, m_ref = 0.5f;
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    if (MODE & 2) {
      tc::tmem_ld32(base + c * 64, v);
      tc::tmem_ld32(base + c * 64 + 32, v + 32);
      tc::tmem_wait_ld();
    } else {
#pragma unroll
      for (int k = 0; k < 64; ++k) v[k] = v[k] * 0.999f;
    }
    uint32_t pk[32];
    const float2 sc2 = make_float2(scale, scale), nmu2 = make_float2(-m_ref, -m_ref);
    float2 la = make_float2(0.f, 0.f), lb = make_float2(0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const float2 xy = __ffma2_rn(make_float2(v[2 * u], v[2 * u + 1]), sc2, nmu2);
      const float2 pp = ((MODE & 4) && (u & 7) == 7) ? poly_exp2x2(xy) : make_float2(fast_exp2(xy.x), fast_exp2(xy.y));
      if (u & 1) lb = __fadd2_rn(lb, pp);
      else la = __fadd2_rn(la, pp);
      pk[u] = pack_bf16(pp.x, pp.y);
    }
    const float ls = (la.x + lb.x) + (la.y + lb.y);
    bool need = !(ls <= 16384.f);
    if (MODE & 1) need = pair_any(1 + quarter + 4 * grp, 64, need);
    else need = __any_sync(0xffffffffu, need);
    if (need) m_ref += 1.f;
    l += ls;
    if ((MODE & 2) && !(MODE & 16)) {
      tc::tmem_stNu<16>(base + 128 + c * 32, pk);
      tc::tmem_stNu<16>(base + 128 + c * 32 + 16, pk + 16);
      tc::tmem_wait_st();
    } else {
      uint32_t x = 0;
#pragma unroll
      for (int u = 0; u < 32; ++u) x ^= pk[u];
      l += __uint_as_float(x & 0x3f000000u);
    }
  }
  long long t1 = clock64();
  if (lane == 0) cyc[warp] = t1 - t0;
  out[threadIdx.x] = l;
  if ((MODE & 8) && !(MODE & 512)) {
    asm volatile("bar.sync 15, %0;" ::"r"((nw - 1) * 32));
    if (threadIdx.x == 0) done_flag = 1;
  }
  tc::fence_before();
  __syncthreads();  // final
  tc::fence_after();
  if (warp == 0) tc::tmem_dealloc(slot, 512);
  (void)nw;
}


// Full-row softmax step (FA4-style: one warp per lane quarter holds whole rows): each warp
// exponentiates its 32 rows x 128 columns per step as two 64-column halves (load, exponentials,
// P store), no cross-warp barrier.  W warps: W / 4 independent rows sets per SMSP.
template <int POLY>
__global__ void __launch_bounds__(512, 1) bench_fullrow(float* out, long long* cyc, float scale) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const int quarter = warp & 3, grp = warp >> 2;  // grp: which S tile (one per warp on the SMSP)
  const uint32_t base = slot + ((uint32_t)(quarter * 32) << 16) + grp * 128;
  {
    float init[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) init[k] = (lane * 7 + k * 13 % 29) * 0.01f - 1.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) tc::tmem_st32(base + c * 32, init);
    tc::tmem_wait_st();
  }
  __syncthreads();
  float l = 0.f, m_ref = 0.5f;
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      float v[64];
      tc::tmem_ld32(base + h * 64, v);
      tc::tmem_ld32(base + h * 64 + 32, v + 32);
      tc::tmem_wait_ld();
      uint32_t pk[32];
      const float2 sc2 = make_float2(scale, scale), nmu2 = make_float2(-m_ref, -m_ref);
      float2 la = make_float2(0.f, 0.f), lb = make_float2(0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const float2 xy = __ffma2_rn(make_float2(v[2 * u], v[2 * u + 1]), sc2, nmu2);
        const float2 pp = (POLY && (u & 7) == 7) ? poly_exp2x2(xy) : make_float2(fast_exp2(xy.x), fast_exp2(xy.y));
        if (u & 1) lb = __fadd2_rn(lb, pp);
        else la = __fadd2_rn(la, pp);
        pk[u] = pack_bf16(pp.x, pp.y);
      }
      const float ls = (la.x + lb.x) + (la.y + lb.y);
      if (__any_sync(0xffffffffu, !(ls <= 16384.f))) m_ref += 1.f;
      l += ls;
      // P of this half -> packed columns [32h, 32h + 32) (S columns < 64h + 64, already read)
      tc::tmem_stNu<16>(base + h * 32, pk);
      tc::tmem_stNu<16>(base + h * 32 + 16, pk + 16);
    }
    tc::tmem_wait_st();
  }
  long long t1 = clock64();
  if (lane == 0) cyc[warp] = t1 - t0;
  out[threadIdx.x] = l;
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(slot, 512);
}

template <int POLY>
void run_fullrow(int warps, const char* name) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 512 * 4);
  cudaMalloc(&cyc, 32 * 8);
  bench_fullrow<POLY><<<1, warps * 32>>>(out, cyc, 0.1275f);
  bench_fullrow<POLY><<<1, warps * 32>>>(out, cyc, 0.1275f);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[32];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
  // per SMSP: warps/4 warps x 4096 elements per step
  printf("%-34s warps/SMSP=%d  %7.1f cyc/step(tile per warp)  %5.2f elem/cyc/SMSP  %s\n", name, warps / 4,
         (double)mx / kIters, (warps / 4) * 4096.0 / ((double)mx / kIters), cudaGetErrorString(e));
  cudaFree(out);
  cudaFree(cyc);
}

template <int MODE>
void run(int warps, const char* name) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 512 * 4);
  cudaMalloc(&cyc, 32 * 8);
  const int threads = (warps + ((MODE & 8) ? 1 : 0)) * 32, sm = (MODE & 8) ? 65536 + 1024 : 0;
  cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  bench<MODE><<<1, threads, sm>>>(out, cyc, 0.1275f);
  bench<MODE><<<1, threads, sm>>>(out, cyc, 0.1275f);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[32];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
  if (MODE & 8) { printf("   per warp:"); for (int w = 0; w < warps; ++w) printf(" %lld", h[w] / kIters); printf("\n"); }
  long long h30 = 0;
  cudaMemcpy(&h30, cyc + 30, 8, cudaMemcpyDeviceToHost);
  if (MODE & 2048) printf("   MMA warp: %lld MMAs in %lld cycles = %.1f cyc/MMA (floor 64)\n", h[31], h30, (double)h30 / h[31]);
  if (MODE & 8) printf("   (tensor: %lld MMAs of 128x128x16 meanwhile = %.0f%% of the window)\n", h[31], 100.0 * h[31] * 64 / mx);
  // per SMSP: warps/4 warps x 2048 elements per step
  printf("%-34s warps/SMSP=%d  %7.1f cyc/step  %5.2f elem/cyc/SMSP  %s\n", name, warps / 4, (double)mx / kIters,
         (warps / 4) * 2048.0 / ((double)mx / kIters), cudaGetErrorString(e));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run_fullrow<1>(4, "full rows, 1 warp/SMSP, poly");
  run_fullrow<1>(8, "full rows, 2 warps/SMSP, poly");
  run_fullrow<0>(4, "full rows, 1 warp/SMSP, MUFU only");
  run<12 | 2048>(8, "regs softmax + pipelined MMA");
  run<14 | 2048>(8, "TMEM softmax + pipelined MMA");
  run<15 | 2048>(8, "TMEM softmax pair bar + pipelined MMA");
  run<12 | 512>(8, "regs, vote, extra warp exits");
  run<12 | 128>(8, "regs, vote, spinner only");
  run<12 | 256>(8, "regs, vote, MMA + nanosleep poll");
  run<14 | 256>(8, "TMEM, vote, MMA + nanosleep poll");
  run<12>(8, "regs, vote, MMA SS+TS");
  run<14>(8, "TMEM ld+st, vote, MMA SS+TS");
  run<14 | 16>(8, "TMEM ld only, vote, MMA SS+TS");
  run<14 | 32>(8, "TMEM ld+st, vote, MMA SS only");
  run<14 | 64>(8, "TMEM ld+st, vote, MMA TS only");
  run<14 | 16 | 32>(8, "TMEM ld only, vote, MMA SS only");
  for (int w : {8}) {
    run<0>(w, "regs only, MUFU only, warp vote");
    run<4>(w, "regs only, +poly, warp vote");
    run<5>(w, "regs only, +poly, pair barrier");
    run<6>(w, "TMEM, +poly, warp vote");
    run<7>(w, "TMEM, +poly, pair barrier (kernel)");
  }
  return 0;
}
