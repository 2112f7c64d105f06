// prefill_tc3.cu — K3 v3: branch-masked prefill, one 128-row query tile per work item with the
// S tile double-buffered in TMEM and the softmax split by columns over two warpgroups.
//
// Why (tools/trace_prefill.py on v2, prefill_tc.cu): with two q tiles per CTA, TMEM holds
// 2 x S + 2 x O = 512 columns, P aliases S, and Q.K^T(j+1) has to queue behind P.V(j); each
// tile's chain was 16 tensor MMAs + a full-row softmax (~3.9k cycles per k step) and the tensor
// core idled a third of the time.  Here TMEM holds three S buffers and one O, so Q.K^T(j+1)
// and Q.K^T(j+2) are issued while the softmax of tile j works, and the softmax of tile j+1
// starts the moment it finishes tile j (with two buffers it still waited on P.V(j-1) + Q.K^T(j+1)
// behind the P(j-1) handoff).  Each row's 128 scores are split over
// two warps of the same TMEM lane quarter (64 columns each): half the per-thread latency,
// both warps of an SMSP pair busy, row max / sum exchanged through shared memory.
//
// Persistent: one CTA per SM pulls (128-row q tile, q head) items from a queue, heaviest
// (last) tiles first.  Roles:
//   warp 0 lane 0: scheduler + TMA for the item's Q tile and the K ring
//   warp 0 lane 1: TMA for the V ring
//   warp 1 lane 0: MMA issuer.  Per item with m processed k tiles (status != 0):
//                    QK(0); QK(1); QK(2); for j: [P(j)] PV(j); QK(j+3)
//                  S(j) = Q.K(j)^T into S buffer j % 3 (SS, M=128 N=128, 8 x K16);
//                  O += P(j).V(j) (TS: P read from TMEM where it overwrote S(j)).
//   warps 2-5 (columns 0-63) and 6-9 (columns 64-127): softmax, thread = row = TMEM lane.
//                  Lazy O rescale (only when the row max grows by > 2^8), after P.V(j-1) is
//                  certified by the V ring's empty barrier.  Epilogue: O / l for its 64 dims.
// Tile lists come from tile_map2: item tile t reads its own list (the k tiles whose status for
// that 128-row tile is not 0, hcount[t] of them; entries keep the pair layout kt | stA << 20 |
// stB << 22, so the status of tile t sits at bit 20 + 2 (t & 1)).
#include <algorithm>
#include <mutex>

#include "tc_common.cuh"

namespace mv {
namespace {

constexpr int kT3 = 128;
constexpr int kQB3 = 2;                // Q tiles (item i uses tile i % kQB3; 3 Q tiles + 2 K slots measured 3% slower)
constexpr int kKSt3 = 5 - kQB3;        // K ring slots (Q tiles + K slots share 5 x 32 KiB)
constexpr int kVSt3 = 2;
constexpr int kThreads3 = 384;   // 12 warps: loader, MMA, 8 softmax, 2 Q rotators
constexpr int kRotWarp0 = 10;
constexpr int kHalf3 = kT3 * 128;  // SW128 half tile: 128 rows x 64 dims
constexpr int kTile3 = 2 * kHalf3;
constexpr int kOffQ3 = 0;  // two Q tiles: item i loads and rotates into tile i & 1
constexpr int kOffK3 = kOffQ3 + kQB3 * kTile3;
constexpr int kOffV3 = kOffK3 + kKSt3 * kTile3;
constexpr int kOffBar3 = kOffV3 + kVSt3 * kTile3;
constexpr int kOffX3 = kOffBar3 + 512;  // row max / sum exchange: [2 parity][2 WG][128 rows] f32
// no alignment slack: the dynamic shared memory base is 1024-aligned here (checked at entry)
constexpr int kSmem3 = kOffX3 + 2 * 2 * 128 * 4;
static_assert(kSmem3 <= 227 * 1024, "prefill v3 smem");
constexpr uint32_t kIdQK3 = tc::idesc_bf16(128, 128, 0, 0);
template <int HD> constexpr uint32_t id_pv3() { return tc::idesc_bf16(128, HD, 0, 1); }
constexpr float kLazy3 = 8.f;
// TMEM columns: three S buffers (S(g) in buffer g % 3) and one O
constexpr int kSB = 2;  // S / P buffers
constexpr uint32_t kS0 = 0, kO0 = kSB * 128;  // O of column half c (all HD dims) at kO0 + c * HD

struct Tc3Params {
  const int32_t* excl;
  const int32_t* hcount;  // [n_qt] processed k tiles per 128-row q tile
  const int32_t* tlist;   // [n_qt][stride] per-tile lists from tile_map2
  const float2* cs;        // [n][64] RoPE (cos, sin) per row and pair, from the K pre-pass
  void* out;
  int out_f32;
  int n, hq, hkv, D, n_qt, stride;
  float scale_log2;
  int n_items;
  int* counters;           // [2] work queue / finished CTAs, in the caller's workspace (zeroed by the RoPE pass)
};

struct __align__(16) Item3 {
  int t, h, m, valid;
  int e0, pad0, pad1, pad2;  // e0: first raw entry of the tile's pair list (read ahead by the scheduler)
};

template <int B, int HD>
__device__ __forceinline__ void qk3(uint64_t qd, uint64_t kd) {
#pragma unroll
  for (int k = 0; k < HD / 16; ++k) {
    const uint64_t off = (uint64_t)(((k >> 2) * kHalf3 + (k & 3) * 32) >> 4);
    tc::mma_ss(kS0 + B * 128, qd + off, kd + off, kIdQK3, k > 0 ? 1u : 0u);
  }
}
// O(h) += P(h) . V[64h, 64h + 64): P of column half h sits in packed columns [64h, 64h + 32)
template <int B, int H, int HD>
__device__ __forceinline__ void pv3(uint64_t vd, bool first) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
    tc::mma_ts(kO0 + H * HD, kS0 + B * 128 + H * 64 + k * 8, vd + (uint64_t)(((H * 4 + k) * 2048) >> 4), id_pv3<HD>(),
               (!first || k > 0) ? 1u : 0u);
}

// every kPolyMod3-th score pair takes poly_exp2x2: 1 pair in 8 gave +2.5% on C3 (16 and 4..6 no better)
constexpr int kPolyMod3 = 8;
// exclusion intervals a softmax thread keeps in registers for its row (nesting depth); deeper ones
// are read from L1 on partial tiles
constexpr int kExvRegs = 4;

__device__ __forceinline__ uint32_t bit_range3(int lo, int hi) {
  lo = max(lo, 0);
  const int w = max(min(hi, 32) - lo, 0);
  uint32_t m;
  asm("bmsk.clamp.b32 %0, %1, %2;" : "=r"(m) : "r"(lo), "r"(w));
  return m;
}
__device__ __forceinline__ void pair_sync(int q) {  // the two softmax warps of lane quarter q
  asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
}
// pair barrier that OR-reduces a predicate over the two softmax warps of lane quarter q
__device__ __forceinline__ bool pair_any(int q, bool pred) {
  uint32_t out;
  asm volatile(
      "{\n.reg .pred pi, po;\nsetp.ne.u32 pi, %1, 0;\nbarrier.cta.red.or.pred po, %2, 64, pi;\nselp.u32 %0, 1, 0, po;\n}\n"
      : "=r"(out)
      : "r"((uint32_t)pred), "r"(1 + q)
      : "memory");
  return out != 0;
}
constexpr float kSumLimit3 = 64.f * 256.f;  // a 64-column half's P mass before the reference must move

template <int HD>
__global__ void __launch_bounds__(kThreads3, 1)
    prefill_tc3_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                       const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_o,
                       Tc3Params P) {
  extern __shared__ uint8_t smem_raw3[];
  uint8_t* smem = smem_align1024(smem_raw3);
  if (smem != smem_raw3) __trap();  // no slack was allocated for alignment
  constexpr int kNH = HD / 64;              // 64-dim SW128 halves per row (head dim 64: one)
  constexpr uint32_t kTileTx = kNH * kHalf3;  // bytes of one Q / K / V tile
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar3);
  uint64_t* q_loaded = bars;             // [kQB3] raw Q tile landed (tx)
  uint64_t* q_full = q_loaded + kQB3;    // [kQB3] Q tile rotated (2 rotator warps)
  uint64_t* q_empty = q_full + kQB3;     // [kQB3] MMA commit after the item's last Q.K^T
  uint64_t* k_full = q_empty + kQB3;     // [kKSt3]
  uint64_t* k_empty = k_full + kKSt3;    // [3]
  uint64_t* v_full = k_empty + kKSt3;    // [2]
  uint64_t* v_empty = v_full + kVSt3;    // [2] MMA commit after P.V (also certifies O for the rescale)
  uint64_t* s_full = v_empty + kVSt3;    // [3] S buffer b written
  uint64_t* p_full = s_full + kSB;       // [kSB][2] the 4 warps of column half h wrote P into S buffer b
  uint64_t* o_fin = p_full + 2 * kSB;    // O final for the item
  uint64_t* o_empty = o_fin + 1;         // epilogue read O (256 threads)
  uint64_t* item_full = o_empty + 1;     // [2]
  uint64_t* slot_empty = item_full + 2;  // [2] V lane + MMA + 8 softmax warps
  uint64_t* qbuf_free = slot_empty + 2;  // [kQB3] the epilogue's output store has read the Q buffer
  uint64_t* stage_full = qbuf_free + kQB3;  // [2] by item parity: the 8 softmax warps staged its output
  static_assert(4 * kQB3 + 2 * kKSt3 + 2 * kVSt3 + 3 * kSB + 8 <= 32, "barrier block");
  Item3* s_item = reinterpret_cast<Item3*>(smem + kOffBar3 + 256);  // after <= 32 barriers, 16 B aligned
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_item + 2);
  float* s_x = reinterpret_cast<float*>(smem + kOffX3);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int b = 0; b < kQB3; ++b) {
      mbar_init(&q_loaded[b], 1);
      mbar_init(&q_full[b], 2);
      mbar_init(&q_empty[b], 1);
      mbar_init(&qbuf_free[b], 1);
    }
    mbar_init(o_fin, 1);
    mbar_init(o_empty, 256);
    mbar_init(&stage_full[0], 8);
    mbar_init(&stage_full[1], 8);
    for (int b = 0; b < kSB; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[2 * b], 128);
      mbar_init(&p_full[2 * b + 1], 128);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&item_full[b], 1);
      mbar_init(&slot_empty[b], 12);  // V lane, MMA, 8 softmax warps, 2 rotator warps
    }
    for (int s = 0; s < kKSt3; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kVSt3; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (*tmem_slot != 0) __trap();  // one CTA per SM owns all 512 columns

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- scheduler + Q / K loader ----------------
      tc::tma_prefetch_desc(&map_q);
      tc::tma_prefetch_desc(&map_k);
      int gk = 0;
      // the next item is claimed (and its count / first list entry loaded) one item ahead, so
      // the queue atomic and the two global loads overlap this item's K loads
      auto claim = [&](Item3& it) {
        const int w = atomicAdd(&P.counters[0], 1);
        it.valid = w < P.n_items;
        it.t = it.valid ? P.n_qt - 1 - w / P.hq : 0;
        it.h = it.valid ? w % P.hq : 0;
        it.m = it.valid ? P.hcount[it.t] : 0;
        it.e0 = it.valid ? P.tlist[(size_t)it.t * P.stride] : 0;
        it.pad0 = it.pad1 = it.pad2 = 0;
      };
      // raw (pre-RoPE) Q tiles go out one item ahead: item i + 1's tile is loaded once item i's first
      // K tiles are out (the buffer held item i - 1's Q and its staged output: q_empty and qbuf_free),
      // so the rotator warps rotate it while item i runs instead of at the item transition
      auto load_q = [&](const Item3& q_it, int qi) {
        const int qb = qi % kQB3;
        if (qi >= kQB3) {
          mbar_wait(&q_empty[qb], ((qi / kQB3) - 1) & 1);
          mbar_wait(&qbuf_free[qb], ((qi / kQB3) - 1) & 1);
        }
        mbar_arrive_expect_tx(&q_loaded[qb], kTileTx);
#pragma unroll
        for (int hh = 0; hh < kNH; ++hh)
          tc::tma_load_3d(smem + kOffQ3 + qb * kTile3 + hh * kHalf3, &map_q, 64 * hh, q_it.h, q_it.t * kT3, &q_loaded[qb]);
      };
      Item3 nxt;
      claim(nxt);
      if (nxt.valid) load_q(nxt, 0);
      for (int i = 0;; ++i) {
        const int buf = i & 1;
        if (i >= 2) mbar_wait(&slot_empty[buf], ((i >> 1) - 1) & 1);
        Item3 it = nxt;
        if (it.valid) claim(nxt);
        it.pad0 = nxt.valid;  // the rotator warps rotate the next item's Q tile during this item
        it.pad1 = nxt.t;
        s_item[buf] = it;
        mbar_arrive(&item_full[buf]);
        if (!it.valid) break;
        const int kvh = it.h / (P.hq / P.hkv);
        const int32_t* lst = P.tlist + (size_t)it.t * P.stride;
        for (int j = 0; j < it.m; ++j) {
          const int e = lst[j];
          const int s = gk % kKSt3;
          if (gk >= kKSt3) mbar_wait(&k_empty[s], ((gk / kKSt3) - 1) & 1);
          const int kt = e & 0xFFFFF;
          mbar_arrive_expect_tx(&k_full[s], kTileTx);
#pragma unroll
          for (int hh = 0; hh < kNH; ++hh)
            tc::tma_load_3d(smem + kOffK3 + s * kTile3 + hh * kHalf3, &map_k, 64 * hh, kvh, kt * kT3, &k_full[s]);
          ++gk;
          if (j == min(kKSt3, it.m) - 1 && nxt.valid) load_q(nxt, i + 1);
        }
        if (it.m == 0 && nxt.valid) load_q(nxt, i + 1);
      }
    } else if (lane == 1) {
      // ---------------- V loader ----------------
      tc::tma_prefetch_desc(&map_v);
      int gv = 0;
      for (int i = 0;; ++i) {
        const int buf = i & 1;
        mbar_wait(&item_full[buf], (i >> 1) & 1);
        const Item3 it = s_item[buf];
        mbar_arrive(&slot_empty[buf]);
        if (!it.valid) break;
        const int kvh = it.h / (P.hq / P.hkv);
        const int32_t* lst = P.tlist + (size_t)it.t * P.stride;
        for (int j = 0; j < it.m; ++j) {
          const int e = lst[j];
          const int s = gv % kVSt3;
          if (gv >= kVSt3) mbar_wait(&v_empty[s], ((gv / kVSt3) - 1) & 1);
          const int kt = e & 0xFFFFF;
          mbar_arrive_expect_tx(&v_full[s], kTileTx);
#pragma unroll
          for (int hh = 0; hh < kNH; ++hh)
            tc::tma_load_3d(smem + kOffV3 + s * kTile3 + hh * kHalf3, &map_v, 64 * hh, kvh, kt * kT3, &v_full[s]);
          ++gv;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // The whole warp runs the issue loop converged (waits, descriptors: warp-uniform values the
    // compiler keeps in uniform registers) and one elected lane issues.  The issuer shares its
    // SMSP with two busy softmax warps, so every instruction per MMA costs issue slots: a
    // lane-0-only loop needed ~11 per MMA (descriptor R2UR + a waterfall per asm) and issued an
    // MMA only every ~100 cycles, under the 64 an M=128 N=128 K=16 MMA takes.
    const uint64_t qd0 = tc::sw128_desc(smem_u32(smem + kOffQ3), 16, 1024);
    const uint64_t kd0 = tc::sw128_desc(smem_u32(smem + kOffK3), 16, 1024);
    const uint64_t vd0 = tc::sw128_desc(smem_u32(smem + kOffV3), kHalf3, 1024);
    int g = 0;  // processed k tiles so far (K/V ring index, S buffer = g % 3)
    auto qk = [&](uint64_t qd, int gg) {  // S(gg % 3) = Q . K(gg)^T
      mbar_wait(&k_full[gg % kKSt3], (gg / kKSt3) & 1);
      tc::fence_after();
      const uint64_t kd = kd0 + (uint64_t)(((gg % kKSt3) * kTile3) >> 4);
      const int b = gg % kSB;
      if (tc::elect_one()) {
        if (b == 0) qk3<0, HD>(qd, kd);
        else qk3<1, HD>(qd, kd);
        tc::mma_commit(&s_full[b]);
        tc::mma_commit(&k_empty[gg % kKSt3]);
      }
      __syncwarp();
    };
    for (int i = 0;; ++i) {
      const int buf = i & 1;
      mbar_wait(&item_full[buf], (i >> 1) & 1);
      const Item3 it = s_item[buf];
      __syncwarp();
      if (lane == 0) mbar_arrive(&slot_empty[buf]);
      if (!it.valid) break;
      const int m = it.m;
      const int qb = i % kQB3;
      const uint64_t qd = qd0 + (uint64_t)((qb * kTile3) >> 4);
      mbar_wait(&q_full[qb], (i / kQB3) & 1);  // rotated by warps 10-11 (generic -> async proxy fenced)
      for (int u = 0; u < kSB && u < m; ++u) qk(qd, g + u);
      if (m <= kSB) {
        if (tc::elect_one()) tc::mma_commit(&q_empty[qb]);
        __syncwarp();
      }
      for (int j = 0; j < m; ++j, ++g) {
        mbar_wait(&v_full[g % kVSt3], (g / kVSt3) & 1);
        const int b = g % kSB;
        if (j == 0 && i >= 1) mbar_wait(o_empty, (i - 1) & 1);  // epilogue of item i-1 read both O
        const uint64_t vd = vd0 + (uint64_t)(((g % kVSt3) * kTile3) >> 4);
        // each column half's P.V goes as soon as its four softmax warps released P
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          mbar_wait(&p_full[2 * b + h], (g / kSB) & 1);
          tc::fence_after();
          if (tc::elect_one()) {
            if (b == 0) {
              if (h == 0) pv3<0, 0, HD>(vd, j == 0);
              else pv3<0, 1, HD>(vd, j == 0);
            } else {
              if (h == 0) pv3<1, 0, HD>(vd, j == 0);
              else pv3<1, 1, HD>(vd, j == 0);
            }
            if (h == 1) tc::mma_commit(&v_empty[g % kVSt3]);
          }
          __syncwarp();
        }
        if (j + kSB < m) {
          qk(qd, g + kSB);  // S buffer g % 2 again: in order behind P.V(g)
          if (j + kSB + 1 == m) {
            if (tc::elect_one()) tc::mma_commit(&q_empty[qb]);
            __syncwarp();
          }
        }
      }
      if (m == 0 && i >= 1) mbar_wait(o_empty, (i - 1) & 1);
      if (tc::elect_one()) tc::mma_commit(o_fin);
      __syncwarp();
    }
  } else if (warp >= kRotWarp0) {
    // ---------------- Q rotators: interleaved RoPE of the raw Q tile, in place ----------------
    // thread = 16-byte chunk (4 dim pairs) of a row; SW128: chunk c of row r sits at c ^ (r & 7)
    // of the row's 128 B in half c >> 3.  Same fp32 arithmetic as the pre-pass (rope_cs values
    // from the per-row table), so rotated Q is bit-identical to rope_qk_kernel's.
    const int rt = threadIdx.x - kRotWarp0 * 32;  // 0..63
    for (int it_i = 0;; ++it_i) {
      const int buf = it_i & 1;
      mbar_wait(&item_full[buf], (it_i >> 1) & 1);
      const Item3 it = s_item[buf];
      __syncwarp();
      if (lane == 0) mbar_arrive(&slot_empty[buf]);
      if (!it.valid) break;
      // item 0's tile first, then (every item) the next item's tile, loaded one item ahead
#pragma unroll 1
      for (int pass = it_i == 0 ? 0 : 1; pass < 2; ++pass) {
      const int qi = it_i + pass;
      if (pass == 1 && !it.pad0) break;
      const int qt_t = pass == 0 ? it.t : it.pad1;
      const int qb = qi % kQB3;
      mbar_wait(&q_loaded[qb], (qi / kQB3) & 1);
      uint8_t* qt = smem + kOffQ3 + qb * kTile3;
      // 32 chunks per thread in 4 batches of 8: all table loads of a batch are in flight together
      constexpr int kBatch = 8;
      constexpr int kCh = HD / 8, kLg = HD == 128 ? 4 : 3;  // 16-byte chunks per row
      for (int b0 = 0; b0 < kT3 * kCh / 64; b0 += kBatch) {
        float4 t01[kBatch], t23[kBatch];
        uint4* q4[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const int ch = rt + 64 * (b0 + u);
          const int row = ch >> kLg, c = ch & (kCh - 1);
          const int grow = min(qt_t * kT3 + row, P.n - 1);  // rows past n are zero-filled: any angle
          q4[u] = reinterpret_cast<uint4*>(qt + (c >> 3) * kHalf3 + row * 128 + (((c & 7) ^ (row & 7)) << 4));
          const float4* tb = reinterpret_cast<const float4*>(P.cs + (size_t)grow * (HD / 2) + c * 4);
          t01[u] = __ldg(tb);
          t23[u] = __ldg(tb + 1);
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          uint4 v = *q4[u];
          __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&v);
          const float cs[4] = {t01[u].x, t01[u].z, t23[u].x, t23[u].z};
          const float sn[4] = {t01[u].y, t01[u].w, t23[u].y, t23[u].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 ab = __bfloat1622float2(h2[j]);
            h2[j] = __floats2bfloat162_rn(ab.x * cs[j] - ab.y * sn[j], ab.x * sn[j] + ab.y * cs[j]);
          }
          *q4[u] = v;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // visible to the tensor core
      __syncwarp();
      if (lane == 0) mbar_arrive(&q_full[qb]);
      }
      // this item's output tile, staged by the softmax warps in its Q buffer: two TMA stores; the
      // buffer returns to the loader once they have read it
      if (warp == kRotWarp0 && lane == 0) {
        mbar_wait(&stage_full[it_i & 1], (it_i >> 1) & 1);
        const int qb_ep = it_i % kQB3;
        if (!P.out_f32) {
          const uint8_t* tile = smem + kOffQ3 + qb_ep * kTile3;
#pragma unroll
          for (int hh = 0; hh < kNH; ++hh)  // rows past n are clipped
            tc::tma_store_3d(&map_o, tile + hh * kHalf3, 64 * hh, it.h, it.t * kT3);
          tc::bulk_commit_group();
          tc::bulk_wait_group_read0();
        }
        mbar_arrive(&qbuf_free[qb_ep]);
      }
      __syncwarp();
    }
    if (warp == kRotWarp0 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores done
  } else {
    // ---------------- softmax: warps 2-5 columns 0-63, warps 6-9 columns 64-127 ----------------
    const int c = (warp - 2) >> 2;      // column half
    const int quarter = warp & 3;       // TMEM lane quarter
    const int r = quarter * 32 + lane;  // row within the tile
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    int g = 0;
    for (int it_i = 0;; ++it_i) {
      const int buf = it_i & 1;
      mbar_wait(&item_full[buf], (it_i >> 1) & 1);
      const Item3 it = s_item[buf];
      __syncwarp();
      if (lane == 0) mbar_arrive(&slot_empty[buf]);
      if (!it.valid) break;
      const int i = it.t * kT3 + r;  // sequence row
      const int2* exr = reinterpret_cast<const int2*>(P.excl) + (size_t)min(i, P.n - 1) * P.D;
      // the row's exclusion intervals, in registers for the whole item (partial tiles only use them)
      int2 exv[kExvRegs];
#pragma unroll
      for (int q = 0; q < kExvRegs; ++q) exv[q] = q < P.D ? __ldg(exr + q) : make_int2(0, 0);
      const int32_t* lst = P.tlist + (size_t)it.t * P.stride;
      const int sh = 20 + 2 * (it.t & 1);
      const uint32_t o_col = kO0 + c * HD;  // this column half's own O (all HD dims)
      float m_ref = -INFINITY, l = 0.f;
      // the list entry of the next tile is loaded one tile ahead (its L2 latency used to sit
      // between releasing P and waiting for the next S)
      // the item's tile list in a register window: lane k holds entry w0 + k, one coalesced load per 32
      // tiles, issued a window ahead (a per-tile load of the next entry stalled ~6% of the softmax samples)
      int win = lane < it.m ? __ldg(lst + lane) : 0;
      int win_next = 32 + lane < it.m ? __ldg(lst + 32 + lane) : 0;
      for (int done = 0; done < it.m; ++done, ++g) {
        if (done > 0 && (done & 31) == 0) {
          win = win_next;
          win_next = done + 32 + lane < it.m ? __ldg(lst + done + 32 + lane) : 0;
        }
        const int e = __shfl_sync(0xffffffffu, win, done & 31);
        const int j0 = (e & 0xFFFFF) * kT3;
        const int status = (e >> sh) & 3;
        const uint32_t s_col = kS0 + (g % kSB) * 128;
        mbar_wait(&s_full[g % kSB], (g / kSB) & 1);
        tc::fence_after();
        float v[64];
        tc::tmem_ld32(lane_base + s_col + c * 64, v);
        tc::tmem_ld32(lane_base + s_col + c * 64 + 32, v + 32);
        tc::tmem_wait_ld();
        if (status != 1) {
          const int lim = min(i, P.n - 1) - j0;  // last visible column
          uint32_t vm[2];
#pragma unroll
          for (int w = 0; w < 2; ++w) vm[w] = bit_range3(0, lim + 1 - (2 * c + w) * 32);
#pragma unroll
          for (int q = 0; q < kExvRegs; ++q) {
            if (q >= P.D) break;
            // branch-free: bit_range3 clamps, so an interval outside this tile clears nothing
            const int a = exv[q].x - j0, b = exv[q].y - j0;
#pragma unroll
            for (int w = 0; w < 2; ++w) vm[w] &= ~bit_range3(a - (2 * c + w) * 32, b - (2 * c + w) * 32);
          }
          for (int q = kExvRegs; q < P.D; ++q) {  // deeper nesting: the rest from memory (L1)
            const int2 e2 = __ldg(exr + q);
            const int a = e2.x - j0, b = e2.y - j0;
#pragma unroll
            for (int w = 0; w < 2; ++w) vm[w] &= ~bit_range3(a - (2 * c + w) * 32, b - (2 * c + w) * 32);
          }
#pragma unroll
          for (int k = 0; k < 64; k += 2) {
            const uint32_t mm = vm[k >> 5] >> (k & 31);
            v[k] = (mm & 1u) ? v[k] : -INFINITY;
            v[k + 1] = (mm & 2u) ? v[k + 1] : -INFINITY;
          }
        }
        uint32_t pk[32];
        auto exps = [&](float mu) {
          // FFMA2 scale, 1 pair in kPolyMod3 on the FMA pipe (relieves the 16/clk/SM MUFU), FADD2 sums
          const float2 sc2 = make_float2(P.scale_log2, P.scale_log2), nmu2 = make_float2(-mu, -mu);
          float2 la = make_float2(0.f, 0.f), lb = make_float2(0.f, 0.f);
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const float2 xy = __ffma2_rn(make_float2(v[2 * u], v[2 * u + 1]), sc2, nmu2);
            const float2 pp = (kPolyMod3 > 0 && (u & 15) % kPolyMod3 == kPolyMod3 - 1)
                                  ? poly_exp2x2(xy)
                                  : make_float2(fast_exp2(xy.x), fast_exp2(xy.y));
            if (u & 1) lb = __fadd2_rn(lb, pp);
            else la = __fadd2_rn(la, pp);
            pk[u] = pack_bf16(pp.x, pp.y);
          }
          return (la.x + lb.x) + (la.y + lb.y);
        };
        // Fast path (no per-tile row max): exponentiate against the row's reference; it moves only on
        // the item's first tile or when this half's mass exceeds kSumLimit3 (every P stays <= 2^14,
        // exact enough in bf16 and far from fp32 overflow).  P of this half goes into this warp's own
        // S columns (packed [64c, 64c + 32)), so it is stored before the OR-reduced pair barrier
        // (the store overlaps the wait); a move rewrites it.
        bool need = m_ref == -INFINITY;
        float ls = 0.f;
        const uint32_t p_col = lane_base + s_col + c * 64;
        if (!__any_sync(0xffffffffu, need)) {
          ls = exps(m_ref);
          need = !(ls <= kSumLimit3);  // also catches inf / NaN sums
          tc::tmem_stNu<16>(p_col, pk);
          tc::tmem_stNu<16>(p_col + 16, pk + 16);
        }
        if (__any_sync(0xffffffffu, need)) {
          // slow path (this warp only: each column half keeps its own reference, sum and O): the
          // max over this half, move the reference, rescale this half's O
          float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
          for (int k = 0; k < 64; k += 2) {
            mx0 = fmaxf(mx0, v[k]);
            mx1 = fmaxf(mx1, v[k + 1]);
          }
          const float mx = fmaxf(mx0, mx1) * P.scale_log2;
          const bool move = m_ref == -INFINITY || mx > m_ref + kLazy3;
          const float nref = move ? fmaxf(m_ref, mx) : m_ref;
          const float alpha = move && m_ref != -INFINITY ? fast_exp2(m_ref - nref) : 1.f;
          if (done >= 1 && __any_sync(0xffffffffu, alpha != 1.f)) {
            // O(c) holds P.V of the previous tile (g - 1): its V slot's release certifies it
            mbar_wait(&v_empty[(g - 1) % kVSt3], ((g - 1) / kVSt3) & 1);
            tc::fence_after();
#pragma unroll 1
            for (int cc = 0; cc < HD / 32; ++cc) {
              float o[32];
              tc::tmem_ld32(lane_base + o_col + cc * 32, o);
              tc::tmem_wait_ld();
#pragma unroll
              for (int k = 0; k < 32; ++k) o[k] *= alpha;
              tc::tmem_st32(lane_base + o_col + cc * 32, o);
            }
          }
          l *= alpha;
          m_ref = nref;
          ls = exps(m_ref == -INFINITY ? 0.f : m_ref);
          tc::tmem_stNu<16>(p_col, pk);
          tc::tmem_stNu<16>(p_col + 16, pk + 16);
        }
        l += ls;
        tc::tmem_wait_st();
        tc::fence_before();
        mbar_arrive(&p_full[2 * (g % kSB) + c]);
      }
      // epilogue: combine the two column halves' (reference, sum, O), exchanged while the last P.V
      // runs; this warp writes dims [c HD/2, (c + 1) HD/2)
      float2* xs2 = reinterpret_cast<float2*>(s_x);
      xs2[c * 128 + r] = make_float2(m_ref, l);
      pair_sync(quarter);
      const float2 ot = xs2[(c ^ 1) * 128 + r];
      pair_sync(quarter);  // both read before the next item's exchange
      const float mm = fmaxf(m_ref, ot.x);
      const float a_me = m_ref == -INFINITY ? 0.f : fast_exp2(m_ref - mm);
      const float a_ot = ot.x == -INFINITY ? 0.f : fast_exp2(ot.x - mm);
      const float lt = l * a_me + ot.y * a_ot;
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
      const float a0 = (c == 0 ? a_me : a_ot) * inv, a1 = (c == 0 ? a_ot : a_me) * inv;
      mbar_wait(o_fin, it_i & 1);
      tc::fence_after();
      // bf16 output: stage the tile in this item's Q buffer (all its Q.K^T completed before o_fin) in
      // the Q tile's SW128 layout; rotator warp 10 writes it with two TMA stores and waits for their
      // reads (~2,500 cycles, off the softmax warps' path).  The per-thread row stores this replaces
      // were 256 uncoalesced wavefronts per warp.  fp32 output: direct row stores.
      const int qb_ep = it_i % kQB3;
#pragma unroll 1
      for (int cc = 0; cc < HD / 64; ++cc) {
        const int d0 = c * (HD / 2) + cc * 32;  // first of the 32 dims of this pass
        uint8_t* stage = smem + kOffQ3 + qb_ep * kTile3 + (d0 >> 6) * kHalf3;
        float o[32], o1[32];
        tc::tmem_ld32(lane_base + kO0 + d0, o);
        tc::tmem_ld32(lane_base + kO0 + HD + d0, o1);
        tc::tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 32; ++k) o[k] = (a0 != 0.f ? o[k] * a0 : 0.f) + (a1 != 0.f ? o1[k] * a1 : 0.f);
        if (!P.out_f32) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int ch = ((d0 & 63) >> 3) + e;  // 16-byte chunk of this row's 128 B half
            *reinterpret_cast<uint4*>(stage + r * 128 + ((ch ^ (r & 7)) << 4)) =
                make_uint4(pack_bf16(o[8 * e], o[8 * e + 1]), pack_bf16(o[8 * e + 2], o[8 * e + 3]),
                           pack_bf16(o[8 * e + 4], o[8 * e + 5]), pack_bf16(o[8 * e + 6], o[8 * e + 7]));
          }
        } else if (i < P.n) {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(P.out) + ((size_t)i * P.hq + it.h) * HD + d0);
#pragma unroll
          for (int e = 0; e < 8; ++e) dst[e] = make_float4(o[4 * e], o[4 * e + 1], o[4 * e + 2], o[4 * e + 3]);
        }
      }
      if (!P.out_f32) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // visible to the TMA
      __syncwarp();
      if (lane == 0) mbar_arrive(&stage_full[it_i & 1]);
      tc::fence_before();
      mbar_arrive(o_empty);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(0, 512);
  }
}

}  // namespace

// v3 launch on rotated q/k and the caller's v; tcount / tlist / hcount from tile_map2.
mv_status prefill_tc3_launch(const __nv_bfloat16* q_raw, const __nv_bfloat16* k_rot, const __nv_bfloat16* v,
                             const float2* cs, const int32_t* d_excl, int32_t max_depth, int32_t n, int32_t q_heads,
                             int32_t kv_heads, int32_t head_dim, void* d_out, int32_t out_dtype, const int32_t* hcount,
                             const int32_t* tlist, int32_t stride, int32_t* counters, cudaStream_t st) {
  if (max_depth > 64) return fail(MV_ERR_INVALID_ARGUMENT, "prefill: max_depth > 64");
  CUtensorMap mq, mk, mvv, mo;
  if (mv_status e = tc::make_rows_map(&mq, q_raw, n, q_heads, kT3, head_dim)) return e;
  // bf16 output map (same [n][hq][128] shape and box as Q); unused for fp32 output
  if (mv_status e = tc::make_rows_map(&mo, out_dtype == 1 ? (const void*)q_raw : d_out, n, q_heads, kT3, head_dim))
    return e;
  if (mv_status e = tc::make_rows_map(&mk, k_rot, n, kv_heads, kT3, head_dim)) return e;
  if (mv_status e = tc::make_rows_map(&mvv, v, n, kv_heads, kT3, head_dim)) return e;
  Tc3Params T;
  T.excl = d_excl;
  T.hcount = hcount;
  T.tlist = tlist;
  T.cs = cs;
  T.out = d_out;
  T.out_f32 = out_dtype == 1;
  T.n = n;
  T.hq = q_heads;
  T.hkv = kv_heads;
  T.D = max_depth;
  T.n_qt = (n + kT3 - 1) / kT3;
  T.stride = stride;
  T.scale_log2 = 1.4426950408889634f / sqrtf((float)head_dim);
  T.n_items = T.n_qt * q_heads;
  static std::once_flag attr_once[kMaxDevices];
  static int sms_dev[kMaxDevices] = {};
  const int cur = current_device();
  cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once[cur], [&] {
    attr_err = cudaDeviceGetAttribute(&sms_dev[cur], cudaDevAttrMultiProcessorCount, cur);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(prefill_tc3_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem3);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(prefill_tc3_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem3);
  });
  MV_CUDA_TRY(attr_err);
  const int num_sms = sms_dev[cur] > 0 ? sms_dev[cur] : 148;
  T.counters = counters;
  if (head_dim == 128) prefill_tc3_kernel<128><<<std::min(T.n_items, num_sms), kThreads3, kSmem3, st>>>(mq, mk, mvv, mo, T);
  else prefill_tc3_kernel<64><<<std::min(T.n_items, num_sms), kThreads3, kSmem3, st>>>(mq, mk, mvv, mo, T);
  MV_LAUNCH_CHECK();
  return MV_OK;
}

}  // namespace mv
