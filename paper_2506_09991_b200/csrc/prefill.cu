// prefill.cu — K3: branch-masked prefill attention over a whole structured sequence.
//
// Reference behaviour replaced: ToyModel::forward (toy_model.cpp:174-202)
// gathers, for every row i, the mask-visible rows j < i and runs the attention core of
// ToyModel::step (toy_model.cpp:121-157) — O(n^2) gathers and scalar fp64 math.  Here the mask
// is the compact interval form produced by K1 (mask[i][j] = j <= i and j outside row i's
// <= D exclusion intervals) and the computation is tiled flash attention:
//   1. rope_qk_kernel: rotate K once at the Multiverse positions (interleaved RoPE) and write a
//      per-row (cos, sin) table for the Q rotation inside the attention kernel.
//   2. tile_map2 (visibility.cu), on a side stream: classify every (128-row q tile, 128-token
//      k tile) as skipped (fully masked cross-branch or above the diagonal), full or partial,
//      and compact per q tile the ordered list of k tiles to process.
//   3. prefill_tc3_kernel (prefill_tc3.cu): persistent tcgen05 / TMEM / TMA flash attention.
#include <map>
#include <mutex>
#include <string>

#include "tc_common.cuh"

namespace mv {
namespace {

constexpr int kMaxD = 64;        // exclusion intervals per row (the first 8 live in registers)

// One thread per (row, 16-byte chunk): the 4 (cos, sin) pairs of the chunk depend only on the
// row's position, so they are computed once and applied to the chunk in every q and k head
// (hq + hkv heads, 256 B apart; a warp covers two rows' 512 contiguous bytes per head).
__global__ void __launch_bounds__(256) rope_qk_kernel(const __nv_bfloat16* __restrict__ q,
                                                      const __nv_bfloat16* __restrict__ k,
                                                      const int32_t* __restrict__ pos, int n, int hq, int hkv,
                                                      const RopeTable rt, __nv_bfloat16* __restrict__ q_rot,
                                                      __nv_bfloat16* __restrict__ k_rot, float2* __restrict__ table,
                                                      int32_t* __restrict__ counters) {
  // re-arm the attention kernel's work queue (it runs after this kernel on the same stream)
  if (counters && blockIdx.x == 0 && threadIdx.x < 2) counters[threadIdx.x] = 0;
  __shared__ double s_inv[kMaxHeadDim / 2];
  const double* inv = rope_stage(rt, s_inv);
  const int hd = rt.hd, lg = hd == 128 ? 4 : 3, ch = 1 << lg;  // 16-byte chunks per head row
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= ((int64_t)n << lg)) return;
  const int row = (int)(x >> lg), c = (int)(x & (ch - 1));
  const int p = __ldg(pos + row);
  float cs[4], sn[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) rope_cs(p, inv[c * 4 + j], cs[j], sn[j]);
  if (table) {  // (cos, sin) per row and pair for the prefill kernel's in-place Q rotation
    float4* tb = reinterpret_cast<float4*>(table + (size_t)row * (hd / 2) + c * 4);
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
  const uint4* qs = reinterpret_cast<const uint4*>(q + (size_t)row * hq * hd) + c;
  uint4* qd = reinterpret_cast<uint4*>(q_rot + (size_t)row * hq * hd) + c;
  // q heads then k heads as one sequence of 16-byte chunks, 8 independent loads in flight
  const uint4* ks = reinterpret_cast<const uint4*>(k + (size_t)row * hkv * hd) + c;
  uint4* kd = reinterpret_cast<uint4*>(k_rot + (size_t)row * hkv * hd) + c;
  const int nq = q_rot ? hq : 0;  // without q_rot only K is rotated (Q rotates in the kernel)
  const int nh = nq + hkv;
  for (int h0 = 0; h0 < nh; h0 += 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int h = h0 + u;
      if (h < nh) v[u] = __ldg(h < nq ? qs + h * ch : ks + (h - nq) * ch);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int h = h0 + u;
      if (h < nh) *(h < nq ? qd + h * ch : kd + (h - nq) * ch) = rot(v[u]);
    }
  }
}

}  // namespace
}  // namespace mv

namespace mv {
mv_status prefill_tc3_launch(const __nv_bfloat16* q_raw, const __nv_bfloat16* k_rot, const __nv_bfloat16* v,
                             const float2* cs, const int32_t* d_excl, int32_t max_depth, int32_t n, int32_t q_heads,
                             int32_t kv_heads, int32_t head_dim, void* d_out, int32_t out_dtype, const int32_t* hcount,
                             const int32_t* tlist, int32_t stride, int32_t* counters, cudaStream_t st);
mv_status tile_map2(const int32_t* d_excl, int32_t n, int32_t max_depth, uint8_t* d_status, int32_t* d_count,
                    int32_t* d_list, int32_t stride, cudaStream_t stream, int32_t* d_hcount, int32_t* d_hlist);
}

using namespace mv;

namespace {

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// Workspace carve-up (all per call: two prefills on different streams share nothing).
struct PrefillWs {
  float2* cs;         // [n][head_dim / 2] RoPE (cos, sin) per row and pair
  __nv_bfloat16* k_rot;  // [n][kv_heads][head_dim]
  int32_t* count;     // [n_qp] pair counts, then [2 n_qp] per-128-row-tile counts
  int32_t* list;      // [n_qp][stride] pair lists, then [2 n_qp][stride] per-tile lists
  uint8_t* status;    // [n_qp][stride] tile statuses
  int32_t* counters;  // [2] work queue / finished CTAs (zeroed by the RoPE pass)
  size_t bytes;
};

PrefillWs carve(void* base, int32_t n, int32_t kv_heads, int32_t hd) {
  const size_t n_qp = (size_t)(n + 255) / 256, stride = (size_t)(n + 127) / 128;
  PrefillWs w;
  uint8_t* p = reinterpret_cast<uint8_t*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    uint8_t* r = p ? p + off : nullptr;
    off += align256(bytes);
    return r;
  };
  w.cs = reinterpret_cast<float2*>(take((size_t)n * (hd / 2) * sizeof(float2)));
  w.k_rot = reinterpret_cast<__nv_bfloat16*>(take((size_t)n * kv_heads * hd * 2));
  w.count = reinterpret_cast<int32_t*>(take(3 * n_qp * 4));
  w.list = reinterpret_cast<int32_t*>(take(3 * n_qp * stride * 4));
  w.status = take(n_qp * stride);
  w.counters = reinterpret_cast<int32_t*>(take(2 * 4));
  w.bytes = off;
  return w;
}

// The tile map (latency-bound, n/256 CTAs) runs on a side stream next to the HBM-bound RoPE pass.
// One side stream and fork/join event pair per (device, caller stream), created once under a lock,
// so concurrent prefills on different streams (or threads) never share one.
struct Side {
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
std::mutex g_side_mu;
std::map<std::pair<int, cudaStream_t>, Side> g_sides;

mv_status side_for(cudaStream_t st, Side* out) {
  std::lock_guard<std::mutex> lk(g_side_mu);
  Side& s = g_sides[{current_device(), st}];
  if (!s.stream) {
    MV_CUDA_TRY(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
    MV_CUDA_TRY(cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming));
    MV_CUDA_TRY(cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming));
  }
  *out = s;
  return MV_OK;
}

}  // namespace

extern "C" size_t mv_prefill_workspace_size_hd(int32_t n, int32_t q_heads, int32_t kv_heads, int32_t head_dim) {
  (void)q_heads;
  return n > 0 && head_dim_supported(head_dim) ? carve(nullptr, n, kv_heads, head_dim).bytes : 0;
}
extern "C" size_t mv_prefill_workspace_size(int32_t n, int32_t q_heads, int32_t kv_heads) {
  return mv_prefill_workspace_size_hd(n, q_heads, kv_heads, kHeadDim);
}

extern "C" mv_status mv_attn_prefill_hd(const void* d_q, const void* d_k, const void* d_v, const int32_t* d_positions,
                                        const int32_t* d_excl, int32_t max_depth, int32_t n, int32_t q_heads,
                                        int32_t kv_heads, int32_t head_dim, double rope_base, void* d_out,
                                        int32_t out_dtype, void* d_workspace, size_t workspace_bytes,
                                        mv_stream_t stream) {
  if (n <= 0) return n == 0 ? MV_OK : fail(MV_ERR_INVALID_ARGUMENT, "mv_attn_prefill: n < 0");
  if (q_heads <= 0 || kv_heads <= 0 || q_heads % kv_heads)
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_attn_prefill: q_heads must be a multiple of kv_heads");
  if (!head_dim_supported(head_dim)) return fail(MV_ERR_INVALID_ARGUMENT, "mv_attn_prefill: head_dim must be 64 or 128");
  if (max_depth < 1 || max_depth > kMaxD)
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_attn_prefill: max_depth in 1.." + std::to_string(kMaxD));
  if (out_dtype != 0 && out_dtype != 1) return fail(MV_ERR_INVALID_ARGUMENT, "out_dtype must be 0 (bf16) or 1 (fp32)");
  if (!d_q || !d_k || !d_v || !d_positions || !d_excl || !d_out || !d_workspace)
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_attn_prefill: null buffer");
  if (workspace_bytes < mv_prefill_workspace_size_hd(n, q_heads, kv_heads, head_dim))
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_attn_prefill: workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const PrefillWs ws = carve(d_workspace, n, kv_heads, head_dim);
  const int n_qp = (n + 255) / 256, stride = (n + 127) / 128;
  int32_t* hcount = ws.count + n_qp;                      // per-128-row-tile counts after the pair counts
  int32_t* hlist = ws.list + (size_t)n_qp * stride;       // per-128-row-tile lists after the pair lists
  Side side;
  if (mv_status e = side_for(st, &side)) return e;
  MV_CUDA_TRY(cudaEventRecord(side.fork, st));
  MV_CUDA_TRY(cudaStreamWaitEvent(side.stream, side.fork, 0));
  if (mv_status e = tile_map2(d_excl, n, max_depth, ws.status, ws.count, ws.list, stride, side.stream, hcount, hlist))
    return e;
  MV_CUDA_TRY(cudaEventRecord(side.join, side.stream));
  // K rotated once; Q is rotated inside the attention kernel from the per-row (cos, sin) table
  rope_qk_kernel<<<(unsigned)(((int64_t)n * (head_dim / 8) + 255) / 256), 256, 0, st>>>(
      (const __nv_bfloat16*)d_q, (const __nv_bfloat16*)d_k, d_positions, n, q_heads, kv_heads,
      make_rope_table(rope_base > 0 ? rope_base : 10000.0, head_dim), nullptr, ws.k_rot, ws.cs, ws.counters);
  MV_LAUNCH_CHECK();
  MV_CUDA_TRY(cudaStreamWaitEvent(st, side.join, 0));
  return prefill_tc3_launch((const __nv_bfloat16*)d_q, ws.k_rot, (const __nv_bfloat16*)d_v, ws.cs, d_excl, max_depth, n,
                            q_heads, kv_heads, head_dim, d_out, out_dtype, hcount, hlist, stride, ws.counters, st);
}

extern "C" mv_status mv_attn_prefill(const void* d_q, const void* d_k, const void* d_v, const int32_t* d_positions,
                                     const int32_t* d_excl, int32_t max_depth, int32_t n, int32_t q_heads,
                                     int32_t kv_heads, double rope_base, void* d_out, int32_t out_dtype,
                                     void* d_workspace, size_t workspace_bytes, mv_stream_t stream) {
  return mv_attn_prefill_hd(d_q, d_k, d_v, d_positions, d_excl, max_depth, n, q_heads, kv_heads, kHeadDim, rope_base,
                            d_out, out_dtype, d_workspace, workspace_bytes, stream);
}
