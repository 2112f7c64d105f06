// common.cuh — shared helpers for the sm_100a kernels (PTX wrappers, status plumbing).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <string>

#include "multiverse_b200.h"

namespace mv {

// Thread-local last-error message behind mv_last_error().
void set_error(const std::string& msg);
mv_status fail(mv_status st, const std::string& msg);

#define MV_CUDA_TRY(expr)                                                                    \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      return ::mv::fail(MV_ERR_CUDA, std::string(#expr " failed: ") + cudaGetErrorString(_e)); \
  } while (0)

#define MV_LAUNCH_CHECK()                                                                          \
  do {                                                                                             \
    cudaError_t _e = cudaGetLastError();                                                           \
    if (_e != cudaSuccess) return ::mv::fail(MV_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(_e)); \
  } while (0)

constexpr int kPageTokens = 16;   // tokens per KV page (BASELINE configs[1] "paged KV block 16")
constexpr int kHeadDim = 128;     // Qwen2.5-32B head dim (BASELINE configs[1..4])
constexpr int kMaxHeadDim = 128;  // head dims with native kernels: 128 and 64 (the toy model's d_h, toy_model.hpp:29)
__host__ __device__ constexpr bool head_dim_supported(int hd) { return hd == 64 || hd == 128; }
constexpr int kTagCount = 10;     // grammar.hpp:47 kTagLiteralCount

// Tag ids (tokenizer.cpp:56-63 / grammar.hpp:34-46).
enum Tag : int32_t {
  kParOpen = 0, kParClose, kGoalOpen, kGoalClose, kOutOpen, kOutClose, kPathOpen, kPathClose, kConcOpen, kConcClose
};

// ---------------------------------------------------------------------------
// Page-table entry: a ragged run of `count` token slots starting at `begin` inside
// `page`. Packed in an int2 so a warp reads 32 entries in one 256 B load.
// ---------------------------------------------------------------------------
struct __align__(8) PageRef {
  int32_t page;
  int32_t bc;  // begin | (count << 8)
};
__host__ __device__ inline int ref_begin(PageRef r) { return r.bc & 0xff; }
__host__ __device__ inline int ref_count(PageRef r) { return (r.bc >> 8) & 0xff; }
__host__ __device__ inline PageRef make_ref(int page, int begin, int count) {
  PageRef r;
  r.page = page;
  r.bc = begin | (count << 8);
  return r;
}

// ---------------------------------------------------------------------------
// KV plane layout (one plane per layer for K, one for V): head-major [kv_head][page][16 x hd block]
//   (hd = head dim, 128 or 64); the block holds token t, dim d at atom (t >> 3, d >> 6) of 1 KiB =
//   8 token rows x 128 B, atoms ordered [t >> 3][d >> 6], 16-byte chunk c of row r stored at chunk
//   c ^ r (SWIZZLE_128B per atom).
// Consecutive page-head blocks of one KV head therefore form canonical UMMA operands with one 1-D bulk
// copy per page: K-major for Q.K^T (N = tokens: 8-row groups hd * 16 B apart, dims 64..127 at +1024 B)
// and MN-major for P.V (N = dims: atoms 1024 B apart, K = tokens: 8-row groups hd * 16 B apart) — no
// shared-memory re-layout.  Head-major: pages p..p+3 of one head are contiguous HBM, so a table block
// of consecutive page ids (bulk allocations hand out ascending runs) is ONE bulk copy.
// ---------------------------------------------------------------------------
__host__ __device__ inline int swz_chunk(int token, int chunk) { return chunk ^ (token & 7); }
// element offset of 16-byte chunk c (dims 8c..8c+7) of token slot t inside a page-head block
__host__ __device__ inline int kv_chunk_offset(int t, int c, int hd) {
  return ((((t >> 3) * (hd >> 6) + (c >> 3)) * 8 + (t & 7)) * 64) + ((((c & 7) ^ (t & 7))) << 3);
}
__host__ __device__ inline size_t kv_page_head_offset(int64_t page, int head, int64_t num_pages, int hd) {
  return ((size_t)head * (size_t)num_pages + (size_t)page) * (size_t)(kPageTokens * hd);
}

// ---------------------------------------------------------------------------
// PTX wrappers (sm_100a)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_n(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// non-blocking probe: has the phase with this parity completed?
// Lazily created per-device state (streams, scratch, function attributes) is indexed by the
// current device, so one process may drive several GPUs.
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < kMaxDevices ? d : kMaxDevices - 1;
}

// Programmatic dependent launch (PDL): the dependent grid may be scheduled once every CTA of
// this grid has called launch_dependents; pdl_wait blocks until the predecessor grid completed
// and its memory is visible (a no-op when the launch carried no programmatic dependency).
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// 1024-byte-aligned view of dynamic shared memory that keeps the shared address space: pointer
// arithmetic on the __shared__ array itself, so data accesses compile to LDS / STS (an integer
// round trip through uintptr_t made them generic LD / ST).
__device__ __forceinline__ uint8_t* smem_align1024(uint8_t* raw) {
  return raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ int ld_volatile_s32(const int* p) {
  int v;
  asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile_s32(int* p, int v) {
  asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

// 1-D bulk copy global -> shared, completing on an mbarrier (TMA engine, no tensor map).
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* gmem, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gmem), "r"(bytes) : "memory");
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                                  uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldmatrix_x2(uint32_t& r0, uint32_t& r1, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ uint32_t movmatrix_trans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

// D(16x8 f32) += A(16x16 bf16, row) * B(16x8 bf16, col)
__device__ __forceinline__ void mma_bf16_16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x for a pair on the FMA pipe (FA4-style MUFU offload): x = j + f with j = rint(x) by the
// 1.5 * 2^23 magic add, 2^f by a degree-3 minimax polynomial on [-0.5, 0.5] (relative error
// 1.1e-4, below bf16's rounding of P), j added into the exponent field.
__device__ __forceinline__ float2 poly_exp2x2(float2 x) {
  // [-126, 64]: keeps j + exponent(p) inside the exponent field (an unclamped x >= 128 wraps into the
  // sign bit and would hide a large score from the callers' softmax sum guards)
  x = make_float2(fminf(fmaxf(x.x, -126.f), 64.f), fminf(fmaxf(x.y, -126.f), 64.f));
  const float2 t = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));
  const float2 j = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __ffma2_rn(j, make_float2(-1.f, -1.f), x);
  float2 p = __ffma2_rn(make_float2(0.05592212f, 0.05592212f), f, make_float2(0.24264069f, 0.24264069f));
  p = __ffma2_rn(p, f, make_float2(0.69312102f, 0.69312102f));
  p = __ffma2_rn(p, f, make_float2(0.99992444f, 0.99992444f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// Interleaved rotary map (toy_model.cpp:30-41): pair t of an hd-dim head rotates by
// theta = pos * base^(-2t/dh). The inverse frequencies are computed on the host with the same
// std::pow expression as the reference, theta is formed and range-reduced in fp64 (positions
// reach 1e5 rad), and only the final sincos runs in fp32.
struct RopeTable {
  double inv[kMaxHeadDim / 2];  // hd / 2 pairs used
  int32_t hd;                   // head dim of the rotated vectors (and of the K/V rows the kernels write)
};
inline RopeTable make_rope_table(double base, int hd) {
  RopeTable t;
  t.hd = hd;
  for (int i = 0; i < kMaxHeadDim / 2; ++i) t.inv[i] = i < hd / 2 ? std::pow(base, -2.0 * (double)i / (double)hd) : 0.0;
  return t;
}
// Stages the frequency table in shared memory.  Indexing the by-value kernel-parameter copy
// with a lane-dependent index serialises in the constant cache (16 distinct addresses per
// warp), which made the RoPE passes ~4x slower than their HBM bound.  Call before any early
// return (it contains a block barrier).
__device__ __forceinline__ const double* rope_stage(const RopeTable& rt, double* s_inv) {
  for (int t = threadIdx.x; t < kMaxHeadDim / 2; t += blockDim.x) s_inv[t] = rt.inv[t];
  __syncthreads();
  return s_inv;
}
__device__ __forceinline__ void rope_cs(int pos, double inv, float& c, float& s) {
  double th = (double)pos * inv;
  th = fma(-6.283185307179586476925286766559, rint(th * 0.15915494309189533576888376337251), th);  // [-pi, pi]
  __sincosf((float)th, &s, &c);  // SFU; |err| < 2^-21 on [-pi, pi]
}

}  // namespace mv
