// prefill_tc.cu — K3 v2: branch-masked prefill on the 5th-gen tensor cores (tcgen05 / TMEM / TMA).
//
// Persistent: one CTA per SM pulls (256-row query pair, q head) items from a queue (heaviest
// pairs first).  The pair is two 128-row tiles A and B that share every K/V tile, so one MMA
// thread can ping-pong between them while two softmax warpgroups work (the FlashAttention-4
// schedule):
//
//   warp 0   lane 0: scheduler + TMA for Q_A, Q_B (once per item) and the K ring; lane 1: V ring
//                   (separate rings: K frees after Q.K^T, V only after P.V)
//   warp 1   MMA  : one thread.  Loop over the pair's listed k tiles j:
//                     PV_A(j); QK_A(j+1); PV_B(j); QK_B(j+1)
//                   S_X = Q_X.K^T (M=128, N=128, 8 x K16, SS operands from SW128 smem) into TMEM;
//                   O_X += P_X.V with P_X read straight from TMEM (TS operand, aliasing S_X).
//                   P arrives in two halves (k tokens 0-63, 64-127) so the first four P.V MMAs
//                   start while the softmax finishes the second half.
//   warps 2-5 softmax A, warps 6-9 softmax B : thread = query row = TMEM lane.  S row by
//                   tcgen05.ld, interval mask on partial tiles (bmsk-built 128-bit row mask),
//                   lazy O rescale in TMEM only when the row max grows by > 2^8, P as packed
//                   bf16 back into the S columns by tcgen05.st (FFMA2 / FADD2 for scale and
//                   row sum).  Epilogue O / l from TMEM.
//
// TMEM (512 columns): S/P_A 0..127, S/P_B 128..255, O_A 256..383, O_B 384..511.
// Ordering facts the schedule relies on: tcgen05.mma ops of one thread execute in issue order,
// so QK_X(j+1) (which overwrites S/P_X) cannot overtake PV_X(j) (which reads P_X), and the
// commit after QK_X(j+1) also certifies PV_X(j) -> the softmax may rescale O_X after s_full.
//
// Measured bound (tools/trace_prefill.py, C3): the per-tile chain is PV_X(j) + QK_X(j+1) on the
// tensor core (16 MMAs at the 64-cycle N=128 tensor rate, ~1.4k cycles) followed by softmax X
// (~2k cycles: 128 MUFU.EX2 per row at 16 lanes/clk/SM, tools/microbench/mb_exp.cu).  S/P
// aliasing (TMEM is full: 2 x S + 2 x O) keeps QK_X(j+1) behind PV_X(j), so the tensor core
// idles ~1/3 of each step.
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

namespace mv {

mv_status tile_map2(const int32_t* d_excl, int32_t n, int32_t max_depth, int32_t* d_count, int32_t* d_list,
                    int32_t stride, cudaStream_t stream, int32_t* d_hcount = nullptr, int32_t* d_hlist = nullptr);

namespace {

constexpr int kT = 128;          // rows per q tile, tokens per k tile
constexpr int kKSt = 3;          // K ring stages
constexpr int kVSt = 2;          // V ring stages
constexpr int kThreads2 = 320;   // 10 warps
constexpr int kHalf2 = kT * 128;  // SW128 half tile (128 rows x 128 B)
constexpr int kTile2 = 2 * kHalf2;
constexpr int kOffQA = 0;
constexpr int kOffQB = kOffQA + kTile2;
constexpr int kOffK2 = kOffQB + kTile2;
constexpr int kOffV2 = kOffK2 + kKSt * kTile2;
constexpr int kOffBar2 = kOffV2 + kVSt * kTile2;
constexpr int kSmem2 = kOffBar2 + 512 + 1024;
constexpr uint32_t kIdQK = tc::idesc_bf16(128, 128, 0, 0);
constexpr uint32_t kIdPV = tc::idesc_bf16(128, 128, 0, 1);
constexpr int kMaxD2 = 8;
constexpr float kLazy2 = 8.f;

struct Tc2Params {
  const int32_t* excl;
  const int32_t* tcount;
  const int32_t* tlist;
  void* out;
  int out_f32;
  int n, hq, hkv, D, n_qp, stride;
  float scale_log2;
  int n_items;          // (q-tile pair, q head) work items, heaviest pairs first
  int* counters;        // [0] work queue, [1] finished CTAs (the last one re-arms the queue)
};

// MMA issue with compile-time TMEM operands (tile X: S/P at column 128X, O at 256 + 128X) and
// descriptors advanced by constants, so the issuing thread does little besides UTCHMMA
template <int X>
__device__ __forceinline__ void pf_qk(uint64_t qd, uint64_t kd) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint64_t off = (uint64_t)(((k >> 2) * kHalf2 + (k & 3) * 32) >> 4);
    tc::mma_ss(X * 128, qd + off, kd + off, kIdQK, k > 0 ? 1u : 0u);
  }
}
// P.V over k tokens [64 H, 64 H + 64): the softmax releases P in two halves so the first four
// MMAs run while it still computes the second half
template <int X, int H>
__device__ __forceinline__ void pf_pv(uint64_t vd, bool first) {
#pragma unroll
  for (int k = 4 * H; k < 4 * H + 4; ++k)
    tc::mma_ts(256 + X * 128, X * 128 + k * 8, vd + (uint64_t)((k * 2048) >> 4), kIdPV, (!first || k > 0) ? 1u : 0u);
}

// bits [lo, hi) of a 32-bit word, lo/hi clamped to [0, 32] (bmsk: one instruction)
__device__ __forceinline__ uint32_t bit_range(int lo, int hi) {
  lo = max(lo, 0);
  const int w = max(min(hi, 32) - lo, 0);
  uint32_t m;
  asm("bmsk.clamp.b32 %0, %1, %2;" : "=r"(m) : "r"(lo), "r"(w));
  return m;
}

struct __align__(16) PfItem {
  int qp, h, cnt, valid;
};

// Persistent: one CTA per SM pulls (q-tile pair, q head) items from a queue and keeps its TMA /
// tensor-core / softmax pipeline running across items (K/V rings, S/P and mbarrier phases
// continue; the next item's Q tile loads while the previous item finishes).
__global__ void __launch_bounds__(kThreads2, 1)
    prefill_tc2_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                       const __grid_constant__ CUtensorMap map_v, Tc2Params P) {
  extern __shared__ uint8_t smem_raw2[];
  uint8_t* smem = smem_align1024(smem_raw2);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar2);
  uint64_t* q_full = bars;                 // Q tiles of the current item landed (tx)
  uint64_t* q_empty = q_full + 1;          // MMA commit: the item's last Q.K^T done -> next Q may land
  uint64_t* k_full = q_empty + 1;
  uint64_t* k_empty = k_full + kKSt;
  uint64_t* v_full = k_empty + kKSt;
  uint64_t* v_empty = v_full + kVSt;
  uint64_t* s_full = v_empty + kVSt;       // [2]: tile A, B
  uint64_t* p_full = s_full + 2;           // [2] P_X columns for k tokens 0-63 written
  uint64_t* p_hi = p_full + 2;             // [2] P_X columns for k tokens 64-127 written
  uint64_t* o_fin = p_hi + 2;              // [2] MMA commit: O_X of the item final
  uint64_t* o_empty = o_fin + 2;           // [2] softmax WG X read O_X (epilogue)
  uint64_t* item_full = o_empty + 2;       // [2] scheduler -> all roles
  uint64_t* slot_empty = item_full + 2;    // [2] V lane + MMA + 8 softmax warps -> scheduler
  PfItem* s_item = reinterpret_cast<PfItem*>(slot_empty + 2);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_item + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < kKSt; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kVSt; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&s_full[x], 1);
      mbar_init(&p_full[x], 128);
      mbar_init(&p_hi[x], 128);
      mbar_init(&o_fin[x], 1);
      mbar_init(&o_empty[x], 128);
      mbar_init(&item_full[x], 1);
      mbar_init(&slot_empty[x], 10);
    }
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  // one CTA per SM allocates all 512 columns, so the base is lane 0 / column 0
  constexpr uint32_t tmem = 0;
  if (*tmem_slot != tmem) __trap();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- scheduler + Q / K loader ----------------
      tc::tma_prefetch_desc(&map_q);
      tc::tma_prefetch_desc(&map_k);
      int gk = 0;
      for (int i = 0;; ++i) {
        const int buf = i & 1;
        if (i >= 2) mbar_wait(&slot_empty[buf], ((i >> 1) - 1) & 1);
        const int w = atomicAdd(&P.counters[0], 1);
        PfItem it;
        it.valid = w < P.n_items;
        it.qp = it.valid ? P.n_qp - 1 - w / P.hq : 0;
        it.h = it.valid ? w % P.hq : 0;
        it.cnt = it.valid ? P.tcount[it.qp] : 0;
        s_item[buf] = it;
        mbar_arrive(&item_full[buf]);
        if (!it.valid) break;
        if (i >= 1) mbar_wait(q_empty, (i - 1) & 1);
        mbar_arrive_expect_tx(q_full, 2 * kTile2);
        tc::tma_load_3d(smem + kOffQA, &map_q, 0, it.h, it.qp * 256, q_full);
        tc::tma_load_3d(smem + kOffQA + kHalf2, &map_q, 64, it.h, it.qp * 256, q_full);
        tc::tma_load_3d(smem + kOffQB, &map_q, 0, it.h, it.qp * 256 + kT, q_full);
        tc::tma_load_3d(smem + kOffQB + kHalf2, &map_q, 64, it.h, it.qp * 256 + kT, q_full);
        const int kvh = it.h / (P.hq / P.hkv);
        const int32_t* lst = P.tlist + (size_t)it.qp * P.stride;
        for (int j = 0; j < it.cnt; ++j, ++gk) {
          const int s = gk % kKSt;
          if (gk >= kKSt) mbar_wait(&k_empty[s], ((gk / kKSt) - 1) & 1);
          const int kt = lst[j] & 0xFFFFF;
          mbar_arrive_expect_tx(&k_full[s], kTile2);
          tc::tma_load_3d(smem + kOffK2 + s * kTile2, &map_k, 0, kvh, kt * kT, &k_full[s]);
          tc::tma_load_3d(smem + kOffK2 + s * kTile2 + kHalf2, &map_k, 64, kvh, kt * kT, &k_full[s]);
        }
      }
    } else if (lane == 1) {
      // ---------------- V loader ----------------
      tc::tma_prefetch_desc(&map_v);
      int gv = 0;
      for (int i = 0;; ++i) {
        const int buf = i & 1;
        mbar_wait(&item_full[buf], (i >> 1) & 1);
        const PfItem it = s_item[buf];
        mbar_arrive(&slot_empty[buf]);
        if (!it.valid) break;
        const int kvh = it.h / (P.hq / P.hkv);
        const int32_t* lst = P.tlist + (size_t)it.qp * P.stride;
        for (int j = 0; j < it.cnt; ++j, ++gv) {
          const int s = gv % kVSt;
          if (gv >= kVSt) mbar_wait(&v_empty[s], ((gv / kVSt) - 1) & 1);
          const int kt = lst[j] & 0xFFFFF;
          mbar_arrive_expect_tx(&v_full[s], kTile2);
          tc::tma_load_3d(smem + kOffV2 + s * kTile2, &map_v, 0, kvh, kt * kT, &v_full[s]);
          tc::tma_load_3d(smem + kOffV2 + s * kTile2 + kHalf2, &map_v, 64, kvh, kt * kT, &v_full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint64_t qdA = tc::sw128_desc(smem_u32(smem + kOffQA), 16, 1024);
      const uint64_t qdB = tc::sw128_desc(smem_u32(smem + kOffQB), 16, 1024);
      const uint64_t kd0 = tc::sw128_desc(smem_u32(smem + kOffK2), 16, 1024);
      const uint64_t vd0 = tc::sw128_desc(smem_u32(smem + kOffV2), kHalf2, 1024);
      auto qk = [&](int x, int g) {  // S_x = Q_x . K(g)^T
        const uint64_t kd = kd0 + (uint64_t)(((g % kKSt) * kTile2) >> 4);
        if (x) pf_qk<1>(qdB, kd);
        else pf_qk<0>(qdA, kd);
        tc::mma_commit(&s_full[x]);
      };
      auto pv = [&](int x, int g, bool first) {  // O_x += P_x(tmem) . V(g), P in two halves
        const uint64_t vd = vd0 + (uint64_t)(((g % kVSt) * kTile2) >> 4);
        if (x) pf_pv<1, 0>(vd, first);
        else pf_pv<0, 0>(vd, first);
        mbar_wait(&p_hi[x], g & 1);
        tc::fence_after();
        if (x) pf_pv<1, 1>(vd, first);
        else pf_pv<0, 1>(vd, first);
      };
      int g = 0;
      for (int i = 0;; ++i) {
        const int buf = i & 1;
        mbar_wait(&item_full[buf], (i >> 1) & 1);
        const PfItem it = s_item[buf];
        mbar_arrive(&slot_empty[buf]);
        if (!it.valid) break;
        mbar_wait(q_full, i & 1);
        const int cnt = it.cnt;
        if (cnt > 0) {
          mbar_wait(&k_full[g % kKSt], (g / kKSt) & 1);
          tc::fence_after();
          qk(0, g);
          qk(1, g);
          tc::mma_commit(&k_empty[g % kKSt]);
          if (cnt == 1) tc::mma_commit(q_empty);
        } else {
          tc::mma_commit(q_empty);
          tc::mma_commit(&o_fin[0]);
          tc::mma_commit(&o_fin[1]);
        }
        for (int j = 0; j < cnt; ++j, ++g) {
          const bool more = j + 1 < cnt;
          mbar_wait(&v_full[g % kVSt], (g / kVSt) & 1);
          mbar_wait(&p_full[0], g & 1);
          if (j == 0 && i >= 1) mbar_wait(&o_empty[0], (i - 1) & 1);  // epilogue drained O_A
          tc::fence_after();
          pv(0, g, j == 0);
          if (more) {
            mbar_wait(&k_full[(g + 1) % kKSt], ((g + 1) / kKSt) & 1);
            tc::fence_after();
            qk(0, g + 1);
          } else {
            tc::mma_commit(&o_fin[0]);
          }
          mbar_wait(&p_full[1], g & 1);
          if (j == 0 && i >= 1) mbar_wait(&o_empty[1], (i - 1) & 1);
          tc::fence_after();
          pv(1, g, j == 0);
          tc::mma_commit(&v_empty[g % kVSt]);
          if (more) {
            qk(1, g + 1);
            tc::mma_commit(&k_empty[(g + 1) % kKSt]);
            if (j + 2 == cnt) tc::mma_commit(q_empty);  // the item's last Q.K^T
          } else {
            tc::mma_commit(&o_fin[1]);
          }
        }
      }
    }
  } else {
    // ---------------- softmax warpgroups: warps 2-5 -> tile A, 6-9 -> tile B ----------------
    const int x = (warp - 2) >> 2;            // tile
    const int quarter = warp & 3;             // TMEM lane quarter this warp may access
    const int r = quarter * 32 + lane;        // row within the tile
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t s_col = x * 128, o_col = 256 + x * 128;
    int gs = 0;
    for (int it_i = 0;; ++it_i) {
      const int buf = it_i & 1;
      mbar_wait(&item_full[buf], (it_i >> 1) & 1);
      const PfItem it = s_item[buf];
      __syncwarp();
      if (lane == 0) mbar_arrive(&slot_empty[buf]);
      if (!it.valid) break;
      const int qp = it.qp, h = it.h, cnt = it.cnt;
      const int32_t* lst = P.tlist + (size_t)qp * P.stride;
      const int i = qp * 256 + x * kT + r;  // sequence row
      // the row's exclusion intervals are re-read (L1) on partial tiles only: keeping 2 x 8 of
      // them in registers next to the 128 scores forced spills
      const int2* exr = reinterpret_cast<const int2*>(P.excl) + (size_t)min(i, P.n - 1) * P.D;
        float m_ref = -INFINITY, l = 0.f;
        for (int j = 0; j < cnt; ++j) {
          const int entry = lst[j];
          const int j0 = (entry & 0xFFFFF) * kT;
          const int status = (entry >> (20 + 2 * x)) & 3;  // 0 skip, 1 full, 2 partial
          mbar_wait(&s_full[x], gs & 1);
          ++gs;
          tc::fence_after();
#if MV_PF_NOSOFT
          if (true) { mbar_arrive(&p_full[x]); mbar_arrive(&p_hi[x]); continue; }
#endif
          float v[kT];
    #pragma unroll
          for (int c = 0; c < 4; ++c) tc::tmem_ld32(lane_base + s_col + c * 32, v + c * 32);
          tc::tmem_wait_ld();
          float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#if MV_PF_NOMASK
          if (false) {
#else
          if (status != 1) {
#endif
            uint32_t vm[4];
            const int lim = status == 0 ? -1 : min(i, P.n - 1) - j0;  // last visible column
    #pragma unroll
            for (int w = 0; w < 4; ++w) vm[w] = bit_range(0, lim + 1 - w * 32);
    #pragma unroll
            for (int q = 0; q < kMaxD2; ++q) {
              if (q >= P.D) break;  // uniform across the CTA
              const int2 ex = __ldg(exr + q);
              const int a = ex.x - j0, e = ex.y - j0;
              if (a >= kT || e <= 0) continue;  // interval misses this k tile
    #pragma unroll
              for (int w = 0; w < 4; ++w) vm[w] &= ~bit_range(a - w * 32, e - w * 32);
            }
    #pragma unroll
            for (int c = 0; c < kT; c += 4) {
              const uint32_t m = vm[c >> 5] >> (c & 31);
              v[c] = (m & 1u) ? v[c] : -INFINITY;
              v[c + 1] = (m & 2u) ? v[c + 1] : -INFINITY;
              v[c + 2] = (m & 4u) ? v[c + 2] : -INFINITY;
              v[c + 3] = (m & 8u) ? v[c + 3] : -INFINITY;
              mx0 = fmaxf(mx0, v[c]); mx1 = fmaxf(mx1, v[c + 1]); mx2 = fmaxf(mx2, v[c + 2]); mx3 = fmaxf(mx3, v[c + 3]);
            }
          } else {
    #pragma unroll
            for (int c = 0; c < kT; c += 4) {
              mx0 = fmaxf(mx0, v[c]); mx1 = fmaxf(mx1, v[c + 1]); mx2 = fmaxf(mx2, v[c + 2]); mx3 = fmaxf(mx3, v[c + 3]);
            }
          }
          // raw-score max; scaled into the log2 domain once (scale > 0 preserves order)
          const float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * P.scale_log2;
          const bool need = mx > m_ref + kLazy2;
          if (__any_sync(0xffffffffu, need)) {
            const float nref = need ? fmaxf(m_ref, mx) : m_ref;
            const float alpha = need ? fast_exp2(m_ref - nref) : 1.f;
            if (j >= 1) {  // s_full(j) certified PV_x(j-1): O_x is final for tiles < j
    #pragma unroll 1
              for (int c = 0; c < 4; ++c) {
                float o[32];
                tc::tmem_ld32(lane_base + o_col + c * 32, o);
                tc::tmem_wait_ld();
    #pragma unroll
                for (int e = 0; e < 32; ++e) o[e] *= alpha;
                tc::tmem_st32(lane_base + o_col + c * 32, o);
              }
            }
            l *= alpha;
            m_ref = nref;
          }
          const float mu = m_ref == -INFINITY ? 0.f : m_ref;
          // packed f32x2 FMA / add (FFMA2, FADD2) halve the scale and row-sum instructions; P
          // (bf16 pairs) overwrites S's first 64 columns 16 packed columns at a time, so only 16
          // packed registers are live next to the 128 scores
          const float2 sc2 = make_float2(P.scale_log2, P.scale_log2), nmu2 = make_float2(-mu, -mu);
          float2 l2 = make_float2(0.f, 0.f), l2b = make_float2(0.f, 0.f);
    #pragma unroll
          for (int c16 = 0; c16 < 4; ++c16) {
            uint32_t pk[16];
    #pragma unroll
            for (int u = 0; u < 16; ++u) {
              const int c = c16 * 16 + u;
              const float2 xy = __ffma2_rn(make_float2(v[2 * c], v[2 * c + 1]), sc2, nmu2);
              const float2 pp = make_float2(fast_exp2(xy.x), fast_exp2(xy.y));
              if (u & 1) l2b = __fadd2_rn(l2b, pp);
              else l2 = __fadd2_rn(l2, pp);
              pk[u] = pack_bf16(pp.x, pp.y);
            }
            tc::tmem_stNu<16>(lane_base + s_col + c16 * 16, pk);
            if (c16 == 1 || c16 == 3) {  // P for k tokens 0-63, then 64-127
              tc::tmem_wait_st();
              tc::fence_before();
              mbar_arrive(c16 == 1 ? &p_full[x] : &p_hi[x]);
            }
          }
          l += (l2.x + l2b.x) + (l2.y + l2b.y);
        }
      // epilogue: O_x / l, then hand O_x back to the MMA issuer
      if (cnt > 0) mbar_wait(&o_fin[x], it_i & 1);
      tc::fence_after();
      const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float o[32];
        tc::tmem_ld32(lane_base + o_col + c * 32, o);
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
      mbar_arrive(&o_empty[x]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(&P.counters[1], 1) == (int)gridDim.x - 1) {
    P.counters[0] = 0;  // every CTA has stopped claiming: re-arm the queue for the next launch
    P.counters[1] = 0;
  }
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

}  // namespace

// Launches the v2 kernel on rotated q/k and the caller's v (all [n][heads][128] bf16).
mv_status prefill_tc2_launch(const __nv_bfloat16* q_rot, const __nv_bfloat16* k_rot, const __nv_bfloat16* v,
                             const int32_t* d_excl, int32_t max_depth, int32_t n, int32_t q_heads, int32_t kv_heads,
                             void* d_out, int32_t out_dtype, int32_t* tcount, int32_t* tlist, cudaStream_t st) {
  if (max_depth > kMaxD2) return fail(MV_ERR_INVALID_ARGUMENT, "prefill: max_depth > 8");
  const int n_qp = (n + 255) / 256;
  const int stride = (n + kT - 1) / kT;
  if (mv_status e = tile_map2(d_excl, n, max_depth, tcount, tlist, stride, st)) return e;
  CUtensorMap mq, mk, mvv;
  if (mv_status e = tc::make_rows_map(&mq, q_rot, n, q_heads, kT)) return e;
  if (mv_status e = tc::make_rows_map(&mk, k_rot, n, kv_heads, kT)) return e;
  if (mv_status e = tc::make_rows_map(&mvv, v, n, kv_heads, kT)) return e;
  Tc2Params T;
  T.excl = d_excl;
  T.tcount = tcount;
  T.tlist = tlist;
  T.out = d_out;
  T.out_f32 = out_dtype == 1;
  T.n = n;
  T.hq = q_heads;
  T.hkv = kv_heads;
  T.D = max_depth;
  T.n_qp = n_qp;
  T.stride = stride;
  T.scale_log2 = 1.4426950408889634f / sqrtf((float)kHeadDim);
  T.n_items = n_qp * q_heads;
  static int* counters_dev[kMaxDevices] = {};
  static int sms_dev[kMaxDevices] = {};
  const int cur = current_device();
  int*& d_counters = counters_dev[cur];
  int& num_sms = sms_dev[cur];
  if (!d_counters) {
    MV_CUDA_TRY(cudaMalloc(&d_counters, 2 * sizeof(int)));
    MV_CUDA_TRY(cudaMemsetAsync(d_counters, 0, 2 * sizeof(int), st));
    int dev = 0;
    MV_CUDA_TRY(cudaGetDevice(&dev));
    MV_CUDA_TRY(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  T.counters = d_counters;
  static bool attr_dev[kMaxDevices] = {};
  if (!attr_dev[cur]) {
    MV_CUDA_TRY(cudaFuncSetAttribute(prefill_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2));
    attr_dev[cur] = true;
  }
  prefill_tc2_kernel<<<std::min(T.n_items, num_sms), kThreads2, kSmem2, st>>>(mq, mk, mvv, T);
  MV_LAUNCH_CHECK();
  return MV_OK;
}

}  // namespace mv
