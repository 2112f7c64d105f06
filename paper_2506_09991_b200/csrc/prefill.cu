// prefill.cu — K3: branch-masked prefill attention over a whole structured sequence.
//
// Reference behaviour replaced: ToyModel::forward (toy_model.cpp:174-202)
// gathers, for every row i, the mask-visible rows j < i and runs the attention core of
// ToyModel::step (toy_model.cpp:121-157) — O(n^2) gathers and scalar fp64 math.  Here the mask
// is the compact interval form produced by K1 (mask[i][j] = j <= i and j outside row i's
// <= D exclusion intervals) and the computation is tiled flash attention:
//   1. rope_qk_kernel: rotate Q and K once at the Multiverse positions (interleaved RoPE).
//   2. mv_tile_map (visibility.cu): classify every (64-row q tile, 64-token k tile) as skipped
//      (fully masked cross-branch or above the diagonal), full, or partial.
//   3. prefill_kernel (v0, mma.sync): one CTA per (q tile, q head), 4 warps x 16 rows; only the
//      listed k tiles are visited, the element mask is evaluated only on partial tiles.
//      K/V tiles stream through a cp.async double buffer (XOR-swizzled rows, conflict-free
//      ldmatrix); S and P stay in registers (FA2 fragment reuse); online softmax in log2 domain.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

namespace mv {
namespace {

constexpr int kBM = 64;          // query rows per CTA
constexpr int kBN = 64;          // key tokens per tile
constexpr int kPfThreads = 128;  // 4 warps x 16 rows
constexpr int kMaxD = 8;         // exclusion intervals per row supported by the kernel

// One thread per (row, 16-byte chunk): the 4 (cos, sin) pairs of the chunk depend only on the
// row's position, so they are computed once and applied to the chunk in every q and k head
// (hq + hkv heads, 256 B apart; a warp covers two rows' 512 contiguous bytes per head).
__global__ void __launch_bounds__(256) rope_qk_kernel(const __nv_bfloat16* __restrict__ q,
                                                      const __nv_bfloat16* __restrict__ k,
                                                      const int32_t* __restrict__ pos, int n, int hq, int hkv,
                                                      const RopeTable rt, __nv_bfloat16* __restrict__ q_rot,
                                                      __nv_bfloat16* __restrict__ k_rot, float2* __restrict__ table) {
  __shared__ double s_inv[kHeadDim / 2];
  const double* inv = rope_stage(rt, s_inv);
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= (int64_t)n * 16) return;
  const int row = (int)(x >> 4), c = (int)(x & 15);
  const int p = __ldg(pos + row);
  float cs[4], sn[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) rope_cs(p, inv[c * 4 + j], cs[j], sn[j]);
  if (table) {  // (cos, sin) per row and pair for the prefill kernel's in-place Q rotation
    float4* tb = reinterpret_cast<float4*>(table + (size_t)row * 64 + c * 4);
    tb[0] = make_float4(cs[0], sn[0], cs[1], sn[1]);
    tb[1] = make_float4(cs[2], sn[2], cs[3], sn[3]);
  }
  auto rot = [&](uint4 v) {
    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 ab = __bfloat1622float2(h2[j]);
      h2[j] = __floats2bfloat162_rn(ab.x * cs[j] - ab.y * sn[j], ab.x * sn[j] + ab.y * cs[j]);
    }
    return v;
  };
  const uint4* qs = reinterpret_cast<const uint4*>(q + (size_t)row * hq * kHeadDim) + c;
  uint4* qd = reinterpret_cast<uint4*>(q_rot + (size_t)row * hq * kHeadDim) + c;
  // q heads then k heads as one sequence of 16-byte chunks, 8 independent loads in flight
  const uint4* ks = reinterpret_cast<const uint4*>(k + (size_t)row * hkv * kHeadDim) + c;
  uint4* kd = reinterpret_cast<uint4*>(k_rot + (size_t)row * hkv * kHeadDim) + c;
  const int nq = q_rot ? hq : 0;  // without q_rot only K is rotated (Q rotates in the kernel)
  const int nh = nq + hkv;
  for (int h0 = 0; h0 < nh; h0 += 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int h = h0 + u;
      if (h < nh) v[u] = __ldg(h < nq ? qs + h * 16 : ks + (h - nq) * 16);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int h = h0 + u;
      if (h < nh) *(h < nq ? qd + h * 16 : kd + (h - nq) * 16) = rot(v[u]);
    }
  }
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(pred ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct PrefillParams {
  const __nv_bfloat16* q;  // rotated [n][hq][128]
  const __nv_bfloat16* k;  // rotated [n][hkv][128]
  const __nv_bfloat16* v;  // [n][hkv][128]
  const int32_t* excl;     // [n][D][2]
  const int32_t* tcount;   // [n_qt]
  const int32_t* tlist;    // [n_qt][n_qt]
  void* out;               // [n][hq][128] bf16 or f32
  int out_f32;
  int n, hq, hkv, D, n_qt;
  float scale_log2;
};

// K or V tile (64 tokens x 128 dims) -> smem rows of 256 B, 16 B chunk c of row r at c ^ (r & 7).
__device__ __forceinline__ void load_tile(uint32_t sbase, const __nv_bfloat16* g, int j0, int n, int hkv, int kvh) {
  for (int x = threadIdx.x; x < kBN * 16; x += kPfThreads) {
    const int r = x >> 4, c = x & 15;
    const int j = j0 + r;
    const bool ok = j < n;
    const __nv_bfloat16* src = g + ((size_t)(ok ? j : 0) * hkv + kvh) * kHeadDim + c * 8;
    cp_async16(sbase + r * 256 + (swz_chunk(r, c) << 4), src, ok);
  }
}

constexpr int kPfSmem = 4 * kBN * 256;  // K and V double buffers (64 KiB, dynamic)

__global__ void __launch_bounds__(kPfThreads) prefill_kernel(PrefillParams P) {
  extern __shared__ __align__(1024) uint8_t pf_smem[];
  uint8_t(*sk)[kBN * 256] = reinterpret_cast<uint8_t(*)[kBN * 256]>(pf_smem);
  uint8_t(*sv)[kBN * 256] = reinterpret_cast<uint8_t(*)[kBN * 256]>(pf_smem + 2 * kBN * 256);
  const int qt = blockIdx.x, h = blockIdx.y;
  const int kvh = h / (P.hq / P.hkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int row0 = qt * kBM + warp * 16;
  const int ra = row0 + g, rb = row0 + g + 8;  // this thread's two rows

  // Q fragments (A operand m16 x k16, row-major): straight from global (read once)
  uint32_t qa[8][4];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    const int d0 = ks * 16 + 2 * t4;
    auto ld = [&](int r, int d) -> uint32_t {
      if (r >= P.n) return 0u;
      return *reinterpret_cast<const uint32_t*>(P.q + ((size_t)r * P.hq + h) * kHeadDim + d);
    };
    qa[ks][0] = ld(ra, d0);
    qa[ks][1] = ld(rb, d0);
    qa[ks][2] = ld(ra, d0 + 8);
    qa[ks][3] = ld(rb, d0 + 8);
  }
  // exclusion intervals of the two rows
  int elo[2][kMaxD], ehi[2][kMaxD];
#pragma unroll
  for (int q = 0; q < kMaxD; ++q) {
    elo[0][q] = ehi[0][q] = elo[1][q] = ehi[1][q] = 0;
    if (q < P.D) {
      if (ra < P.n) { elo[0][q] = P.excl[((size_t)ra * P.D + q) * 2]; ehi[0][q] = P.excl[((size_t)ra * P.D + q) * 2 + 1]; }
      if (rb < P.n) { elo[1][q] = P.excl[((size_t)rb * P.D + q) * 2]; ehi[1][q] = P.excl[((size_t)rb * P.D + q) * 2 + 1]; }
    }
  }

  float o[16][4];
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};

  const int cnt = P.tcount[qt];
  const int32_t* lst = P.tlist + (size_t)qt * P.n_qt;
  if (cnt > 0) {
    const int kt0 = lst[0] & 0xFFFF;
    load_tile(smem_u32(sk[0]), P.k, kt0 * kBN, P.n, P.hkv, kvh);
    load_tile(smem_u32(sv[0]), P.v, kt0 * kBN, P.n, P.hkv, kvh);
    cp_async_commit();
  }
  for (int it = 0; it < cnt; ++it) {
    const int entry = lst[it];
    const int kt = entry & 0xFFFF;
    const bool partial = (entry >> 30) & 1;
    const int buf = it & 1;
    if (it + 1 < cnt) {
      const int kn = lst[it + 1] & 0xFFFF;
      load_tile(smem_u32(sk[buf ^ 1]), P.k, kn * kBN, P.n, P.hkv, kvh);
      load_tile(smem_u32(sv[buf ^ 1]), P.v, kn * kBN, P.n, P.hkv, kvh);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();

    const uint32_t kb = smem_u32(sk[buf]), vb = smem_u32(sv[buf]);
    // S (16 rows x 64 tokens) = Q . K^T
    float s[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {  // two n8 tiles per ldmatrix.x4
        uint32_t b0, b1, b2, b3;
        const int mi = lane >> 3;
        const int tok = np * 16 + (mi >> 1) * 8 + (lane & 7);
        const int chunk = ks * 2 + (mi & 1);
        ldmatrix_x4(b0, b1, b2, b3, kb + tok * 256 + (swz_chunk(tok, chunk) << 4));
        mma_bf16_16816(s[2 * np], qa[ks], b0, b1);
        mma_bf16_16816(s[2 * np + 1], qa[ks], b2, b3);
      }
    }
    // mask + online softmax (rows ra: c0,c1; rb: c2,c3)
    const int j0 = kt * kBN;
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int rr = e >> 1;
        const int j = j0 + nt * 8 + 2 * t4 + (e & 1);
        float x = s[nt][e] * P.scale_log2;
        if (partial) {
          const int i = rr ? rb : ra;
          bool vis = j <= i && j < P.n;
#pragma unroll
          for (int q = 0; q < kMaxD; ++q) vis = vis && !(j >= elo[rr][q] && j < ehi[rr][q]);
          if (!vis) x = -INFINITY;
        }
        s[nt][e] = x;
        mx[rr] = fmaxf(mx[rr], x);
      }
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      mx[rr] = fmaxf(mx[rr], __shfl_xor_sync(0xffffffffu, mx[rr], 1));
      mx[rr] = fmaxf(mx[rr], __shfl_xor_sync(0xffffffffu, mx[rr], 2));
    }
    float al[2], mu[2];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const float mn = fmaxf(m_run[rr], mx[rr]);
      mu[rr] = mn == -INFINITY ? 0.f : mn;
      al[rr] = fast_exp2(m_run[rr] - mu[rr]);
      m_run[rr] = mn;
      l_run[rr] *= al[rr];
    }
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      o[nt][0] *= al[0];
      o[nt][1] *= al[0];
      o[nt][2] *= al[1];
      o[nt][3] *= al[1];
    }
    uint32_t pa[4][4];  // P as A operand (m16 x k16 per 16-token group)
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p0 = fast_exp2(s[nt][0] - mu[0]), p1 = fast_exp2(s[nt][1] - mu[0]);
      const float p2 = fast_exp2(s[nt][2] - mu[1]), p3 = fast_exp2(s[nt][3] - mu[1]);
      l_run[0] += p0 + p1;
      l_run[1] += p2 + p3;
      pa[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(p0, p1);
      pa[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(p2, p3);
    }
    // O (16 rows x 128 dims) += P . V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
      for (int dp = 0; dp < 8; ++dp) {  // two n8 dim tiles per ldmatrix.x4.trans
        uint32_t b0, b1, b2, b3;
        const int mi = lane >> 3;
        const int tok = kk * 16 + (mi & 1) * 8 + (lane & 7);
        const int chunk = dp * 2 + (mi >> 1);
        ldmatrix_x4_trans(b0, b1, b2, b3, vb + tok * 256 + (swz_chunk(tok, chunk) << 4));
        mma_bf16_16816(o[2 * dp], pa[kk], b0, b1);
        mma_bf16_16816(o[2 * dp + 1], pa[kk], b2, b3);
      }
    }
    __syncthreads();  // buffer `buf` is refilled next iteration
  }
  cp_async_wait<0>();

  // finalize: l over the 4 t4-lanes of each row, write O / l
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    l_run[rr] += __shfl_xor_sync(0xffffffffu, l_run[rr], 1);
    l_run[rr] += __shfl_xor_sync(0xffffffffu, l_run[rr], 2);
  }
  const float inv0 = l_run[0] > 0.f ? 1.f / l_run[0] : 0.f, inv1 = l_run[1] > 0.f ? 1.f / l_run[1] : 0.f;
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) {
    const int d = nt * 8 + 2 * t4;
    if (P.out_f32) {
      float* out = reinterpret_cast<float*>(P.out);
      if (ra < P.n) *reinterpret_cast<float2*>(out + ((size_t)ra * P.hq + h) * kHeadDim + d) = make_float2(o[nt][0] * inv0, o[nt][1] * inv0);
      if (rb < P.n) *reinterpret_cast<float2*>(out + ((size_t)rb * P.hq + h) * kHeadDim + d) = make_float2(o[nt][2] * inv1, o[nt][3] * inv1);
    } else {
      __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(P.out);
      if (ra < P.n) *reinterpret_cast<uint32_t*>(out + ((size_t)ra * P.hq + h) * kHeadDim + d) = pack_bf16(o[nt][0] * inv0, o[nt][1] * inv0);
      if (rb < P.n) *reinterpret_cast<uint32_t*>(out + ((size_t)rb * P.hq + h) * kHeadDim + d) = pack_bf16(o[nt][2] * inv1, o[nt][3] * inv1);
    }
  }
}

}  // namespace
}  // namespace mv

namespace mv {
mv_status prefill_tc2_launch(const __nv_bfloat16* q_rot, const __nv_bfloat16* k_rot, const __nv_bfloat16* v,
                             const int32_t* d_excl, int32_t max_depth, int32_t n, int32_t q_heads, int32_t kv_heads,
                             void* d_out, int32_t out_dtype, int32_t* tcount, int32_t* tlist, cudaStream_t st);
mv_status prefill_tc3_launch(const __nv_bfloat16* q_raw, const __nv_bfloat16* k_rot, const __nv_bfloat16* v,
                             const float2* cs, const int32_t* d_excl, int32_t max_depth, int32_t n, int32_t q_heads,
                             int32_t kv_heads, void* d_out, int32_t out_dtype, const int32_t* hcount,
                             const int32_t* tlist, int32_t stride, cudaStream_t st);
mv_status tile_map2(const int32_t* d_excl, int32_t n, int32_t max_depth, int32_t* d_count, int32_t* d_list,
                    int32_t stride, cudaStream_t stream, int32_t* d_hcount, int32_t* d_hlist);
}

using namespace mv;

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

extern "C" size_t mv_prefill_workspace_size(int32_t n, int32_t q_heads, int32_t kv_heads) {
  const size_t n_qt = (size_t)(n + kBM - 1) / kBM;
  // region 1: rotated Q (v0 / v2) or the per-row RoPE (cos, sin) table (v3: n x 64 float2)
  return align256(std::max((size_t)n * q_heads * kHeadDim * 2, (size_t)n * 64 * sizeof(float2))) +
         align256((size_t)n * kv_heads * kHeadDim * 2) +
         align256(n_qt * 4) + align256(n_qt * n_qt * 4) + align256(8);
}

extern "C" mv_status mv_attn_prefill(const void* d_q, const void* d_k, const void* d_v, const int32_t* d_positions,
                                     const int32_t* d_excl, int32_t max_depth, int32_t n, int32_t q_heads,
                                     int32_t kv_heads, double rope_base, void* d_out, int32_t out_dtype,
                                     void* d_workspace, size_t workspace_bytes, mv_stream_t stream) {
  if (n <= 0) return n == 0 ? MV_OK : fail(MV_ERR_INVALID_ARGUMENT, "mv_attn_prefill: n < 0");
  if (q_heads <= 0 || kv_heads <= 0 || q_heads % kv_heads)
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_attn_prefill: q_heads must be a multiple of kv_heads");
  if (max_depth < 1 || max_depth > kMaxD) return fail(MV_ERR_INVALID_ARGUMENT, "mv_attn_prefill: max_depth in 1..8");
  if (out_dtype != 0 && out_dtype != 1) return fail(MV_ERR_INVALID_ARGUMENT, "out_dtype must be 0 (bf16) or 1 (fp32)");
  if (!d_q || !d_k || !d_v || !d_positions || !d_excl || !d_out || !d_workspace)
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_attn_prefill: null buffer");
  if (workspace_bytes < mv_prefill_workspace_size(n, q_heads, kv_heads))
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_attn_prefill: workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int n_qt = (n + kBM - 1) / kBM;
  uint8_t* ws = reinterpret_cast<uint8_t*>(d_workspace);
  __nv_bfloat16* q_rot = reinterpret_cast<__nv_bfloat16*>(ws);
  ws += align256(std::max((size_t)n * q_heads * kHeadDim * 2, (size_t)n * 64 * sizeof(float2)));
  __nv_bfloat16* k_rot = reinterpret_cast<__nv_bfloat16*>(ws);
  ws += align256((size_t)n * kv_heads * kHeadDim * 2);
  int32_t* tcount = reinterpret_cast<int32_t*>(ws);
  ws += align256((size_t)n_qt * 4);
  int32_t* tlist = reinterpret_cast<int32_t*>(ws);
  ws += align256((size_t)n_qt * n_qt * 4);
  unsigned long long* vis = reinterpret_cast<unsigned long long*>(ws);

  const RopeTable rt = make_rope_table(rope_base > 0 ? rope_base : 10000.0);
  const bool v3 = !getenv("MV_PREFILL_V0") && !getenv("MV_PREFILL_TC2");
  const int n_qp = (n + 255) / 256, stride = (n + 127) / 128;
  int32_t* hcount = tcount + n_qp;  // per-128-row-tile processed counts after the n_qp pair counts
  // The tile map (latency-bound, n/256 CTAs) runs on a side stream next to the HBM-bound RoPE
  // pass; the main stream joins it before the attention kernel.
  static cudaStream_t sides[kMaxDevices] = {};
  static cudaEvent_t forks[kMaxDevices] = {}, joins[kMaxDevices] = {};
  const int dev = current_device();
  if (v3 && !sides[dev]) {
    MV_CUDA_TRY(cudaStreamCreateWithFlags(&sides[dev], cudaStreamNonBlocking));
    MV_CUDA_TRY(cudaEventCreateWithFlags(&forks[dev], cudaEventDisableTiming));
    MV_CUDA_TRY(cudaEventCreateWithFlags(&joins[dev], cudaEventDisableTiming));
  }
  cudaStream_t side = sides[dev];
  cudaEvent_t ev_fork = forks[dev], ev_join = joins[dev];
  if (v3) {
    MV_CUDA_TRY(cudaEventRecord(ev_fork, st));
    MV_CUDA_TRY(cudaStreamWaitEvent(side, ev_fork, 0));
    // per-128-row-tile lists after the pair lists (capacity (n/64)^2 >= 3 n^2 / 2^15 entries)
    if (mv_status e = tile_map2(d_excl, n, max_depth, tcount, tlist, stride, side, hcount, tlist + (size_t)n_qp * stride))
      return e;
    MV_CUDA_TRY(cudaEventRecord(ev_join, side));
  }
  // v3 rotates Q in the kernel from a per-row (cos, sin) table (written into the q_rot region)
  float2* cs_table = reinterpret_cast<float2*>(q_rot);
  rope_qk_kernel<<<(unsigned)(((int64_t)n * 16 + 255) / 256), 256, 0, st>>>(
      (const __nv_bfloat16*)d_q, (const __nv_bfloat16*)d_k, d_positions, n, q_heads, kv_heads, rt,
      v3 ? nullptr : q_rot, k_rot, v3 ? cs_table : nullptr);
  MV_LAUNCH_CHECK();

  if (v3) {  // tcgen05 v3 (prefill_tc3.cu)
    MV_CUDA_TRY(cudaStreamWaitEvent(st, ev_join, 0));
    return prefill_tc3_launch((const __nv_bfloat16*)d_q, k_rot, (const __nv_bfloat16*)d_v, cs_table, d_excl, max_depth,
                              n, q_heads, kv_heads, d_out, out_dtype, hcount, tlist + (size_t)n_qp * stride, stride,
                              st);
  }
  MV_CUDA_TRY(cudaMemsetAsync(vis, 0, 8, st));
  if (!getenv("MV_PREFILL_V0"))  // tcgen05 v2 (prefill_tc.cu) and v0 kept for A/B diagnostics
    return prefill_tc2_launch(q_rot, k_rot, (const __nv_bfloat16*)d_v, d_excl, max_depth, n, q_heads, kv_heads, d_out,
                              out_dtype, tcount, tlist, st);
  if (mv_status e = mv_tile_map(d_excl, n, max_depth, kBN, tcount, tlist, vis, stream)) return e;
  PrefillParams P;
  P.q = q_rot;
  P.k = k_rot;
  P.v = (const __nv_bfloat16*)d_v;
  P.excl = d_excl;
  P.tcount = tcount;
  P.tlist = tlist;
  P.out = d_out;
  P.out_f32 = out_dtype == 1;
  P.n = n;
  P.hq = q_heads;
  P.hkv = kv_heads;
  P.D = max_depth;
  P.n_qt = n_qt;
  P.scale_log2 = 1.4426950408889634f / sqrtf((float)kHeadDim);
  static bool attr_set[kMaxDevices] = {};
  if (!attr_set[current_device()]) {
    MV_CUDA_TRY(cudaFuncSetAttribute(prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPfSmem));
    attr_set[current_device()] = true;
  }
  prefill_kernel<<<dim3(n_qt, q_heads), kPfThreads, kPfSmem, st>>>(P);
  MV_LAUNCH_CHECK();
  return MV_OK;
}
