// Throughput of the softmax building blocks on one SM (cycles per warp instruction per SMSP):
// MUFU.EX2, FFMA2, FMNMX3, F2FP pack, and the FMA-pipe poly_exp2.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_exp mb_exp.cu
#include <cstdio>
#include <cuda_bf16.h>

constexpr int kIters = 4096;

template <int MODE>
__global__ void bench(float* out, long long* cyc, float s) {
  float a[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = threadIdx.x * 1e-3f + k * 0.01f - 1.f;
  unsigned acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (MODE == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[k]));
      } else if (MODE == 1) {
        asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(a[k]) : "f"(s));
      } else if (MODE == 2) {
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[k]) : "f"(s), "f"(a[(k + 1) & 15]));
      } else if (MODE == 3) {
        unsigned r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[k]), "f"(a[(k + 1) & 15]));
        acc += r;
      } else if (MODE == 4) {
        asm volatile("add.f32 %0, %0, %1;" : "+f"(a[k]) : "f"(s));
      } else if (MODE == 5) {  // ex2 with only 8 of 32 lanes active (divergent branch)
        if ((threadIdx.x & 31) < 8) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[k]));
      }
    }
  }
  long long t1 = clock64();
  float sum = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) sum += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = sum + acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4096 * 4);
  cudaMalloc(&cyc, 8);
  bench<MODE><<<1, warps * 32>>>(out, cyc, 0.999f);
  bench<MODE><<<1, warps * 32>>>(out, cyc, 0.999f);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double per = (double)c / (kIters * 16.0);  // cycles per instruction per warp
  // warps spread over 4 SMSPs: cycles per warp-instruction per SMSP
  printf("%-10s warps=%2d  %.2f cycles/instr/warp -> %.2f SMSP cycles per warp-instr (%.1f lanes/clk/SM)\n", name, warps,
         per, per / ((warps + 3) / 4), 32.0 * warps / per);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("ex2", w);
    run<1>("ffma", w);
    run<2>("fmnmx3", w);
    run<3>("f2fp", w);
    run<4>("fadd", w);
    run<5>("ex2 8/32", w);
  }
  return 0;
}
