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
#include <cstdlib>

#include "tc_common.cuh"

namespace mv {
namespace {

constexpr int kBM = 64;          // query rows per CTA
constexpr int kBN = 64;          // key tokens per tile
constexpr int kPfThreads = 128;  // 4 warps x 16 rows
constexpr int kMaxD = 8;         // exclusion intervals per row supported by the kernel
constexpr float kLazyRescalePf = 8.f;  // log2-domain headroom before O is rescaled

__global__ void rope_qk_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                               const int32_t* __restrict__ pos, int n, int hq, int hkv, const RopeTable rt,
                               __nv_bfloat16* __restrict__ q_rot, __nv_bfloat16* __restrict__ k_rot) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // one 16 B chunk (4 pairs)
  const int64_t nq = (int64_t)n * hq * 16, nk = (int64_t)n * hkv * 16;
  if (x >= nq + nk) return;
  const bool isq = x < nq;
  const int64_t y = isq ? x : x - nq;
  const int c = (int)(y & 15);
  const int row = (int)(y / (16 * (isq ? hq : hkv)));
  const __nv_bfloat16* src = isq ? q : k;
  __nv_bfloat16* dst = isq ? q_rot : k_rot;
  uint4 v = *reinterpret_cast<const uint4*>(src + y * 8);
  __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&v);
  const int p = pos[row];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float cs, sn;
    rope_cs(p, rt.inv[c * 4 + j], cs, sn);
    const float2 ab = __bfloat1622float2(h2[j]);
    h2[j] = __floats2bfloat162_rn(ab.x * cs - ab.y * sn, ab.x * sn + ab.y * cs);
  }
  *reinterpret_cast<uint4*>(dst + y * 8) = v;
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

// ===========================================================================
// v1: tcgen05 / TMEM / TMA kernel (one CTA per (128-row q tile, q head))
// ===========================================================================
//   warp 0      TMA: Q tile once, then K and V tiles of every listed k tile into a 2-stage ring
//               (SW128 K-major halves via 3-D tensor maps; OOB rows zero-filled).
//   warp 1      MMA (one thread): S[b] = Q.K^T (M=128, N=128, 8 x K16) into TMEM, double-
//               buffered, then O += P.V (P from smem K-major, V MN-major) one tile behind.
//   warps 4-7   softmax: thread = query row = TMEM lane; S row via tcgen05.ld, interval mask on
//               partial tiles, lazy O rescale in TMEM (only when the row max grows by > 2^8),
//               P as bf16 into SW128 smem; epilogue O / l straight from TMEM.
constexpr int kTM = 128, kTN = 128;
constexpr int kTcStages = 2;
constexpr int kTcThreads = 256;
constexpr int kHalf = kTM * 128;                      // one SW128 half tile: 128 rows x 128 B
constexpr int kTile = 2 * kHalf;                      // 32 KiB
constexpr int kOffQ = 0;
constexpr int kOffK = kOffQ + kTile;
constexpr int kOffV = kOffK + kTcStages * kTile;
constexpr int kOffP = kOffV + kTcStages * kTile;
constexpr int kOffBarTc = kOffP + 2 * kTile;
constexpr int kTcSmem = kOffBarTc + 256 + 1024;       // barriers + alignment slack
constexpr uint32_t kIdescQK = tc::idesc_bf16(128, 128, 0, 0);
constexpr uint32_t kIdescPV = tc::idesc_bf16(128, 128, 0, 1);

struct TcParams {
  const int32_t* excl;
  const int32_t* tcount;
  const int32_t* tlist;
  void* out;
  int out_f32;
  int n, hq, hkv, D, n_qt;
  float scale_log2;
};

__global__ void __launch_bounds__(kTcThreads, 1)
    prefill_tc_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                      const __grid_constant__ CUtensorMap map_v, TcParams P) {
  extern __shared__ uint8_t tc_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBarTc);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + kTcStages;
  uint64_t* s_full = kv_empty + kTcStages;
  uint64_t* s_free = s_full + 2;
  uint64_t* p_full = s_free + 2;
  uint64_t* p_free = p_full + 2;
  uint64_t* o_done = p_free + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 1);

  const int qt = P.n_qt - 1 - blockIdx.x;  // heaviest (late) q tiles first
  const int h = blockIdx.y;
  const int kvh = h / (P.hq / P.hkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cnt = P.tcount[qt];
  const int32_t* lst = P.tlist + (size_t)qt * P.n_qt;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_free[b], 128);
      mbar_init(&p_full[b], 128);
      mbar_init(&p_free[b], 1);
    }
    mbar_init(o_done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch_desc(&map_q);
      tc::tma_prefetch_desc(&map_k);
      tc::tma_prefetch_desc(&map_v);
      mbar_arrive_expect_tx(q_full, kTile);
      tc::tma_load_3d(smem + kOffQ, &map_q, 0, h, qt * kTM, q_full);
      tc::tma_load_3d(smem + kOffQ + kHalf, &map_q, 64, h, qt * kTM, q_full);
      for (int it = 0; it < cnt; ++it) {
        const int s = it % kTcStages;
        if (it >= kTcStages) mbar_wait(&kv_empty[s], ((it / kTcStages) - 1) & 1);
        const int kt = lst[it] & 0xFFFF;
        mbar_arrive_expect_tx(&kv_full[s], 2 * kTile);
        uint8_t* kd = smem + kOffK + s * kTile;
        uint8_t* vd = smem + kOffV + s * kTile;
        tc::tma_load_3d(kd, &map_k, 0, kvh, kt * kTN, &kv_full[s]);
        tc::tma_load_3d(kd + kHalf, &map_k, 64, kvh, kt * kTN, &kv_full[s]);
        tc::tma_load_3d(vd, &map_v, 0, kvh, kt * kTN, &kv_full[s]);
        tc::tma_load_3d(vd + kHalf, &map_v, 64, kvh, kt * kTN, &kv_full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t q_base = smem_u32(smem + kOffQ);
      auto pv = [&](int j) {
        const int b = j & 1, s = j % kTcStages;
        mbar_wait(&p_full[b], (j >> 1) & 1);
        tc::fence_after();
        const uint32_t p_base = smem_u32(smem + kOffP + b * kTile);
        const uint32_t v_base = smem_u32(smem + kOffV + s * kTile);
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // 16 tokens per MMA
          const uint64_t ad = tc::sw128_desc(p_base + (k >> 2) * kHalf + (k & 3) * 32, 16, 1024);
          const uint64_t bd = tc::sw128_desc(v_base + k * 2048, kHalf, 1024);
          tc::mma_ss(tmem + 256, ad, bd, kIdescPV, (j > 0 || k > 0) ? 1u : 0u);
        }
        tc::mma_commit(&p_free[b]);
        tc::mma_commit(&kv_empty[s]);
        tc::mma_commit(o_done);
      };
      mbar_wait(q_full, 0);
      tc::fence_after();
      for (int it = 0; it < cnt; ++it) {
        const int b = it & 1, s = it % kTcStages;
        mbar_wait(&kv_full[s], (it / kTcStages) & 1);
        if (it >= 2) mbar_wait(&s_free[b], ((it >> 1) - 1) & 1);
        tc::fence_after();
        const uint32_t k_base = smem_u32(smem + kOffK + s * kTile);
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // 16 dims per MMA
          const uint32_t off = (k >> 2) * kHalf + (k & 3) * 32;
          const uint64_t ad = tc::sw128_desc(q_base + off, 16, 1024);
          const uint64_t bd = tc::sw128_desc(k_base + off, 16, 1024);
          tc::mma_ss(tmem + b * 128, ad, bd, kIdescQK, k > 0 ? 1u : 0u);
        }
        tc::mma_commit(&s_full[b]);
        if (it >= 1) pv(it - 1);
      }
      if (cnt > 0) pv(cnt - 1);
    }
  } else if (warp >= 4) {
    // ---------------- softmax warpgroup: one query row per thread ----------------
    const int r = (warp - 4) * 32 + lane;
    const int i = qt * kTM + r;
    const uint32_t lane_addr = tmem + ((uint32_t)((warp - 4) * 32) << 16);
    int elo[kMaxD], ehi[kMaxD];
#pragma unroll
    for (int q = 0; q < kMaxD; ++q) {
      elo[q] = ehi[q] = 0;
      if (q < P.D && i < P.n) {
        elo[q] = P.excl[((size_t)i * P.D + q) * 2];
        ehi[q] = P.excl[((size_t)i * P.D + q) * 2 + 1];
      }
    }
    float m_ref = -INFINITY, l = 0.f;
    for (int it = 0; it < cnt; ++it) {
      const int b = it & 1;
      const int entry = lst[it];
      const int j0 = (entry & 0xFFFF) * kTN;
      const bool partial = (entry >> 30) & 1;
      mbar_wait(&s_full[b], (it >> 1) & 1);
      tc::fence_after();
      float x[kTN];
#pragma unroll
      for (int c = 0; c < 4; ++c) tc::tmem_ld32(lane_addr + b * 128 + c * 32, x + c * 32);
      tc::tmem_wait_ld();
      tc::fence_before();
      mbar_arrive(&s_free[b]);
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < kTN; ++c) {
        float v = x[c] * P.scale_log2;
        if (partial) {
          const int j = j0 + c;
          bool vis = j <= i && j < P.n;
#pragma unroll
          for (int q = 0; q < kMaxD; ++q) vis = vis && !(j >= elo[q] && j < ehi[q]);
          if (!vis) v = -INFINITY;
        }
        x[c] = v;
        mx = fmaxf(mx, v);
      }
      const bool need = mx > m_ref + kLazyRescalePf;
      if (__any_sync(0xffffffffu, need)) {
        const float nref = need ? fmaxf(m_ref, mx) : m_ref;
        const float alpha = need ? fast_exp2(m_ref - nref) : 1.f;  // m_ref = -inf -> 0 (O is still 0)
        if (it >= 1) {
          mbar_wait(o_done, (it - 1) & 1);  // PV(it-1) has landed in O
          tc::fence_after();
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            float o[32];
            tc::tmem_ld32(lane_addr + 256 + c * 32, o);
            tc::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] *= alpha;
            tc::tmem_st32(lane_addr + 256 + c * 32, o);
          }
          tc::tmem_wait_st();
        }
        l *= alpha;
        m_ref = nref;
      }
      const float mu = m_ref == -INFINITY ? 0.f : m_ref;
      if (it >= 2) mbar_wait(&p_free[b], ((it >> 1) - 1) & 1);
      uint8_t* prow = smem + kOffP + b * kTile + r * 128;
#pragma unroll
      for (int c = 0; c < 16; ++c) {  // 8 tokens per 16 B chunk
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float p0 = fast_exp2(x[c * 8 + 2 * e] - mu), p1 = fast_exp2(x[c * 8 + 2 * e + 1] - mu);
          l += p0 + p1;
          w[e] = pack_bf16(p0, p1);
        }
        const int half = c >> 3, ch = c & 7;
        *reinterpret_cast<uint4*>(prow + half * kHalf + ((ch ^ (r & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      tc::fence_proxy_async();
      mbar_arrive(&p_full[b]);
    }
    // epilogue: O / l from TMEM
    // s_full(cnt-1) already implied PV(cnt-3) landed; step through the last two o_done phases so a
    // parity wait can never match an older phase.
    if (cnt >= 2) mbar_wait(o_done, (cnt - 2) & 1);
    if (cnt >= 1) mbar_wait(o_done, (cnt - 1) & 1);
    tc::fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      float o[32];
      tc::tmem_ld32(lane_addr + 256 + c * 32, o);
      tc::tmem_wait_ld();
      if (i < P.n) {
        if (P.out_f32) {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(P.out) + ((size_t)i * P.hq + h) * kHeadDim + c * 32);
#pragma unroll
          for (int e = 0; e < 8; ++e) dst[e] = make_float4(o[4 * e] * inv, o[4 * e + 1] * inv, o[4 * e + 2] * inv, o[4 * e + 3] * inv);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(P.out) + ((size_t)i * P.hq + h) * kHeadDim + c * 32);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            dst[e] = make_uint4(pack_bf16(o[8 * e] * inv, o[8 * e + 1] * inv), pack_bf16(o[8 * e + 2] * inv, o[8 * e + 3] * inv),
                                pack_bf16(o[8 * e + 4] * inv, o[8 * e + 5] * inv), pack_bf16(o[8 * e + 6] * inv, o[8 * e + 7] * inv));
        }
      }
    }
    tc::fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

}  // namespace
}  // namespace mv

using namespace mv;

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

extern "C" size_t mv_prefill_workspace_size(int32_t n, int32_t q_heads, int32_t kv_heads) {
  const size_t n_qt = (size_t)(n + kBM - 1) / kBM;
  return align256((size_t)n * q_heads * kHeadDim * 2) + align256((size_t)n * kv_heads * kHeadDim * 2) +
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
  ws += align256((size_t)n * q_heads * kHeadDim * 2);
  __nv_bfloat16* k_rot = reinterpret_cast<__nv_bfloat16*>(ws);
  ws += align256((size_t)n * kv_heads * kHeadDim * 2);
  int32_t* tcount = reinterpret_cast<int32_t*>(ws);
  ws += align256((size_t)n_qt * 4);
  int32_t* tlist = reinterpret_cast<int32_t*>(ws);
  ws += align256((size_t)n_qt * n_qt * 4);
  unsigned long long* vis = reinterpret_cast<unsigned long long*>(ws);

  const RopeTable rt = make_rope_table(rope_base > 0 ? rope_base : 10000.0);
  const int64_t chunks = (int64_t)n * (q_heads + kv_heads) * 16;
  rope_qk_kernel<<<(unsigned)((chunks + 255) / 256), 256, 0, st>>>(
      (const __nv_bfloat16*)d_q, (const __nv_bfloat16*)d_k, d_positions, n, q_heads, kv_heads, rt, q_rot, k_rot);
  MV_LAUNCH_CHECK();
  MV_CUDA_TRY(cudaMemsetAsync(vis, 0, 8, st));

  if (!getenv("MV_PREFILL_V0")) {
    // v1: tcgen05 path (tile map at 128)
    const int n_qt128 = (n + kTM - 1) / kTM;
    if (mv_status e = mv_tile_map(d_excl, n, max_depth, kTN, tcount, tlist, vis, stream)) return e;
    CUtensorMap mq, mk, mvv;
    if (mv_status e = tc::make_rows_map(&mq, q_rot, n, q_heads, kTM)) return e;
    if (mv_status e = tc::make_rows_map(&mk, k_rot, n, kv_heads, kTN)) return e;
    if (mv_status e = tc::make_rows_map(&mvv, d_v, n, kv_heads, kTN)) return e;
    TcParams T;
    T.excl = d_excl;
    T.tcount = tcount;
    T.tlist = tlist;
    T.out = d_out;
    T.out_f32 = out_dtype == 1;
    T.n = n;
    T.hq = q_heads;
    T.hkv = kv_heads;
    T.D = max_depth;
    T.n_qt = n_qt128;
    T.scale_log2 = 1.4426950408889634f / sqrtf((float)kHeadDim);
    static bool tc_attr = false;
    if (!tc_attr) {
      MV_CUDA_TRY(cudaFuncSetAttribute(prefill_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem));
      tc_attr = true;
    }
    prefill_tc_kernel<<<dim3(n_qt128, q_heads), kTcThreads, kTcSmem, st>>>(mq, mk, mvv, T);
    MV_LAUNCH_CHECK();
    return MV_OK;
  }
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
  static bool attr_set = false;
  if (!attr_set) {
    MV_CUDA_TRY(cudaFuncSetAttribute(prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPfSmem));
    attr_set = true;
  }
  prefill_kernel<<<dim3(n_qt, q_heads), kPfThreads, kPfSmem, st>>>(P);
  MV_LAUNCH_CHECK();
  return MV_OK;
}
