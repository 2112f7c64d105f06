// decode.cu — K4: branch-parallel paged decode attention on the 5th-gen tensor cores
// (tcgen05 / TMEM, 1-D TMA bulk copies), split-KV with cascade over the fork lineage.
//
// Reference behaviour replaced: for every active lane the
// engine resolves the lane's whole context (engine.cpp:603-605) and runs the attention core
// of ToyModel::step (toy_model.cpp:121-157): scores q.k/sqrt(dh) over the context in layout
// order, max-subtract, exp, sum, weighted V sum.  Here all lanes of all requests run in one
// launch and the shared Map prefix is read from HBM once per group of sibling branches.
//
// Plan (host, cached per page-table shape): every decoding handle's table is cut at its fork
// lineage boundaries; the segment [prev boundary, boundary of group g) is identical in all
// holders of g, so it becomes ONE cascade unit whose query rows are all holders x GQA heads.
// Segments are split into chunks of up to 256 pages (split-KV, >= 1.5 waves of units); a work
// unit = (chunk, <= 16 handles, KV head), ordered longest-first for the persistent scheduler;
// units of 33-64 rows carry a second row copy in the idle lane quadrants.
//
// Kernel: persistent, one CTA per SM, 16 warps, dynamic work queue (re-armed by the last CTA),
// launched programmatically dependent on rope_q_tile_kernel.
//   warp 0  stager  : claims the next unit, stages its page entries (the TMA lanes may start
//                     streaming), then bulk-copies the members' RoPE'd Q rows (pre-swizzled by
//                     rope_q_tile_kernel; the first copy waits on griddepcontrol) into the Q tile.
//   warp 1  TMA     : lanes 0-7 K, lanes 8-15 V; two 4-lane groups per stream, lane p of a group
//                     copies page p of a 4-page block (1-D bulk copies of the page-head blocks,
//                     already in UMMA SWIZZLE_128B layout in HBM, common.cuh) into 5 K / 6 V ring
//                     slots (mbarrier complete_tx).  Runs ahead across work units.
//   warp 3  QK      : one thread.  Per unit: Q smem -> TMEM (tcgen05.cp).  Per block:
//                     S = Q.K_blk^T (M=128 query rows, N=64 tokens, K=128; A = Q from TMEM) into
//                     one of 3 TMEM S buffers.
//   warp 2  PV      : one thread.  After the softmax, per page O += P_page.V_page (TS: P read
//                     from TMEM, aliasing S; N=128 dims).
//   warps 4-11 softmax: thread = query row = TMEM lane; the two warps of a lane quadrant split
//                     each block's columns and share the row's reference max (barrier-reduced).
//                     Masks ragged page slots, log2-domain softmax against a lazily moved
//                     reference (no per-block max), one score pair in four on the FMA pipe,
//                     P as packed bf16 back into TMEM.
//   warps 12-15 epilogue: O is double-buffered by unit parity (TMEM: 3 S + 2 O + Q = 512 columns), so the
//                     epilogue of unit i drains O[i & 1] while unit i + 1 accumulates into the other.
//                     Sums row copies; O row from TMEM -> final output (single-chunk
//                     handles) or an fp32 split-KV partial, merged afterwards by combine_kernel
//                     (log-sum-exp over the handle's chunks, one CTA per (handle, q head)).
// Query rows: member m of a unit owns TMEM lanes [m*R, m*R + gqa), R = gqa rounded up to a
// power of two >= 8, so every member's rows share the swizzle phase and a 1 KiB-aligned slot.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "store.hpp"
#include "tc_common.cuh"

namespace mv {

namespace {

constexpr int kThreads = 512;                               // 16 warps
// Warp w issues on SM sub-partition w % 4, shared with softmax / epilogue warps of TMEM lane
// quadrant w % 4.  Query rows fill quadrants from 0, so the latency-critical MMA issuers sit on
// sub-partitions 3 (QK) and 2 (PV), idle unless a unit has > 64 rows.
constexpr int kWarpStage = 0, kWarpTma = 1, kWarpPv = 2, kWarpQk = 3;
constexpr int kPageBytes = kPageTokens * kHeadDim * 2;      // 4 KiB page-head block at head dim 128 (ring slots are sized
                                                            // for it; head dim 64 fills half of each slot / Q tile)
template <int HD> constexpr int page_bytes() { return kPageTokens * HD * 2; }
constexpr int kBlkPages = 4;                                // pages per block (one QK MMA chain)
constexpr int kBlkCols = kBlkPages * kPageTokens;           // 64 S columns per block
constexpr int kKSlots = 5, kVSlots = 6;                     // K / V rings, one block (4 pages) per slot (5/6 measured best against 4/7, 6/5, 3/8)
constexpr int kSlotBytes = kBlkPages * kPageBytes;          // 4 page-head blocks as stored (16 KiB)
constexpr int kMaxChunk = 256;                              // split-KV chunk cap (pages); the planner halves it down to 64-16 when work is scarce
constexpr int kMaxEntries = kMaxChunk + 16;                 // pages per work unit (a tail chunk grows in place)
constexpr int kMaxMem = 16;                                 // handles per work unit
constexpr int kQHalf = 128 * 128;                           // [128 rows][64 dims] bf16
constexpr int kQBytes = 2 * kQHalf;
constexpr float kSumLimit = 4096.f;                        // block mass that moves the softmax reference
constexpr int kSBufs = 3;                                   // S / P buffers in flight (3 leaves room for two O)
// every kDecPoly-th score pair on the FMA pipe: C2 +4.5% (1/8: +2.4%, 1/3 ~ 1/4, 1/2 no gain);
// C4: 1/2 -3.5%, 1/3 -0.5%, 1/6 -2%
constexpr int kDecPoly = 4;
constexpr int kTmaLanesPerBlkGroup = 2;  // 4-lane copy groups per stream (blocks in flight per step): C2 +1.4% over 1
constexpr int kColS = 0;                                    // TMEM: S0..S2 (64 cols each)
constexpr int kColO = kSBufs * kBlkCols;                    //       O of even / odd units (2 x 128 cols)
constexpr int kColQ = kColO + 2 * 128;                      //       Q (64 cols: 128 bf16 dims)
static_assert(kColQ + 64 <= 512, "TMEM budget");
constexpr int kTmemCols = 512;

struct __align__(16) WorkItem {
  int64_t entry_off;             // absolute arena index of the chunk's first entry
  int32_t n_entries;             // pages (1..64)
  int32_t n_mem;                 // handles sharing the chunk
  int32_t slot_base;             // partial slot of member 0 (member m -> slot_base + m)
  int32_t kvh;                   // KV head
  int32_t valid;
  int32_t copies;                // query-row copies F (1, 2, 4): rows replicated across lane quadrants
  int32_t members[kMaxMem];      // batch indices
};
static_assert(sizeof(WorkItem) == 96, "WorkItem layout");
constexpr int kItemInts = sizeof(WorkItem) / 4;

constexpr int kOffQ = 0;
constexpr int kOffRing = kOffQ + kQBytes;  // one Q staging tile: TMEM holds the live copy
constexpr int kOffVRing = kOffRing + kKSlots * kSlotBytes;
constexpr int kOffEnt = kOffVRing + kVSlots * kSlotBytes;
constexpr int kOffItem = kOffEnt + 2 * kMaxEntries * 8;
constexpr int kOffEp = kOffItem + 2 * sizeof(WorkItem);
constexpr int kOffStat = kOffEp + 2 * sizeof(WorkItem);
// (reference, sum) per unit parity, warp half, row
constexpr int kOffFlag = kOffStat + 2 * 2 * 128 * 8;  // softmax group max exchange: QPC x NP x 32 = 256 floats for every F
constexpr int kOffRag = kOffFlag + 256 * 4;           // per item buffer: bit b = block b has a ragged page [2][4] words
constexpr int kRagWords = (kMaxEntries / kBlkPages + 31) / 32;
static_assert(kRagWords <= 4, "ragged-block bitmask");
constexpr int kOffXch = kOffRag + 2 * 4 * 4;          // epilogue copy merge [3][32][16] floats
constexpr int kOffBar = kOffXch + 3 * 32 * 16 * 4;
constexpr int kNumBars = 4 + 2 * (kKSlots + kVSlots) + 3 * kSBufs + 7 + 2;
constexpr int kOffTmem = kOffBar + kNumBars * 8;
// no alignment slack: with no static shared memory the dynamic base is 1024-aligned (checked at entry)
constexpr int kSmem = kOffTmem + 16;
static_assert(kSmem <= 227 * 1024, "decode smem");

constexpr uint32_t kIdQK = tc::idesc_bf16(128, kBlkCols, 0, 0);  // S(128 x 64) = Q . K_blk^T
template <int HD> constexpr uint32_t id_pv() { return tc::idesc_bf16(128, HD, 0, 1); }  // O(128 x HD) += P_page . V_page

struct DecodeParams {
  const PageRef* arena;
  const __nv_bfloat16* kplane;
  const __nv_bfloat16* vplane;
  const __nv_bfloat16* q_tile;  // [n][kv_heads][HD / 64][R][64] RoPE'd, swizzled (rope_q_tile_kernel)
  const WorkItem* units;
  int n_units;
  int* work_counter;
  float* part_o;                // [slots][q_heads][128]
  float2* part_ml;              // [slots][q_heads] (log2-domain reference max, sum)
  const int32_t* slot_cnt;      // [n] partial slots per handle
  const int32_t* slot_ptr;      // [n + 1]
  const int32_t* slot_idx;
  void* out;
  int out_f32;
  int kv_heads, q_heads, gqa, R;
  int64_t num_pages;             // page pool size (head stride of the planes)
  float scale_log2;
};

template <int HD>
__device__ __forceinline__ void store_row(const DecodeParams& P, int64_t row, int c, const float* o, float inv) {
  if (P.out_f32) {
    float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(P.out) + row * HD + c * 32);
#pragma unroll
    for (int e = 0; e < 8; ++e) dst[e] = make_float4(o[4 * e] * inv, o[4 * e + 1] * inv, o[4 * e + 2] * inv, o[4 * e + 3] * inv);
  } else {
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(P.out) + row * HD + c * 32);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      dst[e] = make_uint4(pack_bf16(o[8 * e] * inv, o[8 * e + 1] * inv), pack_bf16(o[8 * e + 2] * inv, o[8 * e + 3] * inv),
                          pack_bf16(o[8 * e + 4] * inv, o[8 * e + 5] * inv), pack_bf16(o[8 * e + 6] * inv, o[8 * e + 7] * inv));
  }
}

// MMA issue helpers with compile-time TMEM operands: the issuing thread then needs no per-MMA
// register -> uniform-register moves (which the compiler otherwise wraps in an ELECT loop).
template <int HD>
__device__ __forceinline__ void store_row16(const DecodeParams& P, int64_t row, int k, const float* o, float inv) {
  if (P.out_f32) {
    float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(P.out) + row * HD + k * 16);
#pragma unroll
    for (int e = 0; e < 4; ++e) dst[e] = make_float4(o[4 * e] * inv, o[4 * e + 1] * inv, o[4 * e + 2] * inv, o[4 * e + 3] * inv);
  } else {
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(P.out) + row * HD + k * 16);
#pragma unroll
    for (int e = 0; e < 2; ++e)
      dst[e] = make_uint4(pack_bf16(o[8 * e] * inv, o[8 * e + 1] * inv), pack_bf16(o[8 * e + 2] * inv, o[8 * e + 3] * inv),
                          pack_bf16(o[8 * e + 4] * inv, o[8 * e + 5] * inv), pack_bf16(o[8 * e + 6] * inv, o[8 * e + 7] * inv));
  }
}

template <int SB, int HD>
__device__ __forceinline__ void issue_qk_mmas(uint64_t kd) {  // S_SB = Q . K_blk^T (A = Q in TMEM), HD / 16 K-steps
#pragma unroll
  for (int k = 0; k < HD / 16; ++k)
    tc::mma_ts(kColS + SB * kBlkCols, kColQ + k * 8, kd + (uint64_t)(((k >> 2) * 1024 + (k & 3) * 32) >> 4), kIdQK,
               k > 0 ? 1u : 0u);
}
// P of a block: each softmax part (W = 64 / (2F) tokens) is packed into the first W / 2 of its own
// S columns, so page k's 16 tokens sit at packed column (k >> 1) * 32 + (k & 1) * 8 (F = 1) or
// k * 16 (F = 2)
template <int SB, int HD>
__device__ __forceinline__ void issue_pv_mmas(uint64_t vd, int np, uint32_t acc0, int copies, uint32_t ocol) {  // O += P_SB . V_blk
  constexpr uint32_t pcol = kColS + SB * kBlkCols, id = id_pv<HD>();
  constexpr int pb = page_bytes<HD>();
  const uint32_t p1 = copies == 1 ? 8 : 16, p2 = 32, p3 = copies == 1 ? 40 : 48;
  tc::mma_ts(ocol, pcol, vd, id, acc0);
  if (np > 1) tc::mma_ts(ocol, pcol + p1, vd + (uint64_t)(pb >> 4), id, 1u);
  if (np > 2) tc::mma_ts(ocol, pcol + p2, vd + (uint64_t)((2 * pb) >> 4), id, 1u);
  if (np > 3) tc::mma_ts(ocol, pcol + p3, vd + (uint64_t)((3 * pb) >> 4), id, 1u);
}
// named barrier over the softmax warps holding one logical row quadrant, OR-reducing a predicate
__device__ __forceinline__ bool group_any(int id, int count, bool pred) {
  uint32_t out;
  asm volatile(
      "{\n.reg .pred pi, po;\nsetp.ne.u32 pi, %1, 0;\nbarrier.cta.red.or.pred po, %2, %3, pi;\nselp.u32 %0, 1, 0, po;\n}\n"
      : "=r"(out)
      : "r"((uint32_t)pred), "r"(id), "r"(count)
      : "memory");
  return out != 0;
}
__device__ __forceinline__ void group_sync(int id, int count) {
  asm volatile("barrier.cta.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// One work unit of the softmax role for one warp (F = query-row copies).  Thread = TMEM lane.
// Copy c of the unit's rows lives in lane quadrants [c * 4/F, (c+1) * 4/F); the block's 64
// token columns are split into 2F parts: copy c, warp half h owns part 2c + h and writes zeros
// into the other copies' parts of its rows, so every copy accumulates a disjoint slice of the
// tokens into its own O rows (summed by the epilogue).  All 2F warps holding a logical row share
// its reference max through one named barrier per block (OR-reduced "move" flag).
template <int F, int HD>
__device__ __forceinline__ void softmax_unit(const DecodeParams& P, int& g, int n_ent, int n_mem,
                                             const PageRef* se, const uint32_t* rag, int warp, int lane, uint32_t tmem,
                                             uint64_t* s_full,
                                             uint64_t* p_full, uint64_t* vempty, float* xmax, float& m_out,
                                             float& l_out, int ob) {
  constexpr int QPC = 4 / F, RPC = 32 * QPC, NP = 2 * F, W = kBlkCols / NP, WP = W / 2;
  const int q = warp & 3, half = (warp - 4) >> 2;
  const int c = q / QPC, lq = q % QPC;
  const int r = q * 32 + lane, lr = r - c * RPC;
  const int mi = lr / P.R, hl = lr % P.R;
  const bool row_active = mi < n_mem && hl < P.gqa;
  const bool warp_active = lq * 32 < n_mem * P.R;  // uniform over the group
  const int part = c * 2 + half;
  const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
  const uint32_t ocol = lane_base + kColO + ob * 128 + half * (HD / 2);  // this warp half rescales HD / 2 O columns
  float* gmax = xmax + lq * (NP * 32);
  // named barrier per (copy layout, row quadrant group): units with different F never share an
  // id, so warps that run ahead into the next unit (inactive ones skip barriers) cannot mix
  // arrivals of differently sized barriers (ids 2-5: F = 1, 6-7: F = 2, 8: F = 4; 1: epilogue)
  const int bar_id = (F == 1 ? 2 : (F == 2 ? 6 : 8)) + lq, bar_cnt = 64 * F;
  const int nblk = (n_ent + kBlkPages - 1) / kBlkPages;
  const uint32_t rg0 = rag[0], rg1 = rag[1], rg2 = rag[2], rg3 = rag[3];  // ragged-block bits in registers
  float m_ref = -INFINITY, l = 0.f;
  for (int blk = 0; blk < nblk; ++blk, ++g) {
    const int sb = g % kSBufs;
    const uint32_t scol = lane_base + kColS + sb * kBlkCols;
    mbar_wait(&s_full[sb], (g / kSBufs) & 1);
    tc::fence_after();
    if (warp_active) {
      float v[W];
      tc::tmem_ldN<W>(scol + part * W, v);
      // valid slots of this part's tokens (ragged unit head / tail pages, partial pages)
      const int t0 = part * W;
      constexpr uint32_t kFull = W == 32 ? 0xFFFFFFFFu : ((1u << W) - 1u);
      // padding rows (GQA heads past gqa, lanes past the unit's members) take no mask: their exponentials
      // run against an infinite reference (P = 0), so only a ragged page costs the select below
      uint32_t vm = row_active ? 0u : kFull;
      const uint32_t rw = blk < 32 ? rg0 : (blk < 64 ? rg1 : (blk < 96 ? rg2 : rg3));
      if (row_active && !((rw >> (blk & 31)) & 1u)) vm = kFull;  // every page of the block full
      if (vm != kFull) {
#pragma unroll
        for (int p = 0; p < (W + 15) / 16; ++p) {
          const int pg = blk * kBlkPages + t0 / 16 + p;
          if (pg < n_ent) {
            const PageRef ref = se[pg];
            const uint32_t pm = ((1u << ref_count(ref)) - 1u) << ref_begin(ref);
            vm |= (W == 8 ? (pm >> (t0 & 15)) & 0xFFu : pm) << (16 * p);
          }
        }
      }
      tc::tmem_wait_ld();
      if (!__all_sync(0xffffffffu, vm == kFull)) {
#pragma unroll
        for (int t = 0; t < W; ++t) v[t] = ((vm >> t) & 1u) ? v[t] : -INFINITY;
      }
      uint32_t pk[WP];
      auto exp_part = [&](float mu) {
        // FFMA2 scale, one score pair in kDecPoly on the FMA pipe (poly_exp2x2: the MUFU at
        // 16 lanes/clk/SM bounds the softmax of wide cascade units), FADD2 row sums
        const float2 sc2 = make_float2(P.scale_log2, P.scale_log2), nmu2 = make_float2(-mu, -mu);
        float2 la = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < WP; ++k) {
          const float2 xy = __ffma2_rn(make_float2(v[2 * k], v[2 * k + 1]), sc2, nmu2);
          const float2 pp = (kDecPoly > 0 && k % kDecPoly == kDecPoly - 1)
                                ? poly_exp2x2(xy)
                                : make_float2(fast_exp2(xy.x), fast_exp2(xy.y));
          la = __fadd2_rn(la, pp);
          pk[k] = pack_bf16(pp.x, pp.y);
        }
        return la.x + la.y;
      };
      // Fast path: exponentiate against the row's shared reference; it moves only on the unit's
      // first block or when a part's mass exceeds kSumLimit / NP (P stays exact enough in bf16
      // and far from fp32 overflow), so no per-block max is needed.
      bool need = row_active && m_ref == -INFINITY;
      float ls = 0.f;
      // P of this part goes into its own S columns (packed [part W, part W + W/2)), the zeros into
      // the other copies' parts of these rows: no warp's store touches S another warp still reads,
      // so they are issued before the group barrier (which only decides a reference move)
      if (F > 1) {
        uint32_t z[WP];
#pragma unroll
        for (int k = 0; k < WP; ++k) z[k] = 0u;
#pragma unroll
        for (int c2 = 0; c2 < F; ++c2)
          if (c2 != c) tc::tmem_stNu<WP>(scol + (c2 * 2 + half) * W, z);
      }
      if (!__any_sync(0xffffffffu, need)) {
        ls = exp_part(row_active ? m_ref : INFINITY);
        need = ls > kSumLimit / NP;
        tc::tmem_stNu<WP>(scol + part * W, pk);
      }
      if (group_any(bar_id, bar_cnt, need)) {
        // slow path (whole group): row max over all parts, move the reference, rescale O
        float mx = -INFINITY;
#pragma unroll
        for (int t = 0; t < W; ++t) mx = fmaxf(mx, v[t]);
        gmax[part * 32 + lane] = mx;
        group_sync(bar_id, bar_cnt);
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) mx = fmaxf(mx, gmax[pp * 32 + lane]);
        mx *= P.scale_log2;  // raw-score max into the log2 domain (scale > 0 keeps order)
        group_sync(bar_id, bar_cnt);  // all read before the next exchange overwrites
        const bool move = row_active && (m_ref == -INFINITY || mx > m_ref + 8.f);
        const float nref = move ? mx : m_ref;
        const bool resc = move && m_ref != -INFINITY;
        const float alpha = resc ? fast_exp2(m_ref - nref) : 1.f;
        if (blk > 0 && __any_sync(0xffffffffu, resc)) {
          // O holds blocks < blk of this unit once PV(g-1) has completed (its V slot commit)
          mbar_wait(&vempty[(g - 1) % kVSlots], ((g - 1) / kVSlots) & 1);
          tc::fence_after();
#pragma unroll 1
          for (int cc = 0; cc < HD / 64; ++cc) {
            float o[32];
            tc::tmem_ld32(ocol + cc * 32, o);
            tc::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] *= alpha;
            tc::tmem_st32(ocol + cc * 32, o);
          }
        }
        l *= alpha;
        m_ref = nref;
        ls = exp_part(!row_active ? INFINITY : (m_ref == -INFINITY ? 0.f : m_ref));
        tc::tmem_stNu<WP>(scol + part * W, pk);
      }
      l += ls;
      tc::tmem_wait_st();
    }
    tc::fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&p_full[sb]);
  }
  m_out = m_ref;
  l_out = l;
}
template <int HD>
__device__ __forceinline__ void issue_q_copy(uint64_t qd) {  // Q tile smem -> TMEM (HD / 64 halves)
#pragma unroll
  for (int k = 0; k < HD / 16; ++k) tc::cp_128x256b(kColQ + k * 8, qd + (uint64_t)(((k >> 2) * kQHalf + (k & 3) * 32) >> 4));
}

template <int HD>
__global__ void __launch_bounds__(kThreads, 1) decode_tc_kernel(const DecodeParams P) {
  constexpr int kNH = HD / 64;                // Q / K / V 64-dim atoms per row
  constexpr int kPB = page_bytes<HD>();       // page-head block bytes
  constexpr int kRunBytes = kBlkPages * kPB;  // a 4-page block of consecutive pages
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  if (smem != smem_raw) __trap();  // no slack was allocated for alignment
  uint8_t* ring = smem + kOffRing;
  WorkItem* s_item = reinterpret_cast<WorkItem*>(smem + kOffItem);
  WorkItem* s_ep = reinterpret_cast<WorkItem*>(smem + kOffEp);
  PageRef* s_ent0 = reinterpret_cast<PageRef*>(smem + kOffEnt);
  float2* s_stat = reinterpret_cast<float2*>(smem + kOffStat);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* item_full = bars;             // [2] stager -> TMA / MMA / softmax (count 1 + Q tx)
  uint64_t* slot_empty = bars + 2;        // [2] TMA + MMA commit + 8 softmax warps -> stager
  uint64_t* kfull = bars + 4;             // [kKSlots] TMA -> QK issuer
  uint64_t* kempty = kfull + kKSlots;     // [kKSlots] QK commit -> TMA
  uint64_t* vfull = kempty + kKSlots;     // [kVSlots] TMA -> PV issuer
  uint64_t* vempty = vfull + kVSlots;     // [kVSlots] PV commit -> TMA (and softmax O rescale)
  uint64_t* s_full = vempty + kVSlots;    // [kSBufs] QK commit -> softmax
  uint64_t* p_full = s_full + kSBufs;     // [kSBufs] 8 softmax warps -> PV issuer
  uint64_t* pv_done = p_full + kSBufs;    // [kSBufs] PV commit -> QK issuer (S buffer free)
  // O is double-buffered by unit parity: unit i accumulates into O[i & 1] while the epilogue drains unit i - 1
  uint64_t* o_full = pv_done + kSBufs;    // [2] PV commit -> epilogue (unit's O final)
  uint64_t* o_empty = o_full + 2;         // [2] epilogue warps -> PV issuer / softmax (O, stats, header read)
  uint64_t* stat_full = o_empty + 2;      // [2] 8 softmax warps -> epilogue
  uint64_t* q_free = stat_full + 2;       // QK issuer commit (Q tile copied to TMEM) -> stager
  uint64_t* ent_full = q_free + 1;        // [2] stager -> TMA lanes: header + page entries staged (no Q)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffTmem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ent_full[b], 1);
      mbar_init(&item_full[b], 1);
      mbar_init(&slot_empty[b], 12);  // 2 TMA lanes + QK commit + PV issuer + 8 softmax warps
    }
    for (int b = 0; b < kSBufs; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 8);
      mbar_init(&pv_done[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&o_full[b], 1);
      mbar_init(&o_empty[b], 4);
      mbar_init(&stat_full[b], 8);
    }
    mbar_init(q_free, 1);
    for (int s = 0; s < kKSlots; ++s) {
      mbar_init(&kfull[s], 1);
      mbar_init(&kempty[s], 1);
    }
    for (int s = 0; s < kVSlots; ++s) {
      mbar_init(&vfull[s], 1);
      mbar_init(&vempty[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == kWarpQk) tc::tmem_alloc(tmem_slot, kTmemCols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  // One CTA per SM allocates all 512 columns, so the allocation starts at lane 0 / column 0.  A
  // compile-time base keeps every TMEM operand uniform (no per-MMA R2UR waterfall in the issuer).
  constexpr uint32_t tmem = 0;
  if (*tmem_slot != tmem) __trap();
  // programmatic launch: everything but the Q tile (written by rope_q_tile_kernel, the kernel
  // this one may overlap) is ready, so only the stager waits (before its first Q copy); the page
  // tables and K/V planes were final before rope_q_tile_kernel started
  pdl_launch_dependents();

  if (warp == kWarpStage) {
    // ---------------- stager: claim, entries, Q rows ----------------
    int w_next = lane == 0 ? atomicAdd(P.work_counter, 1) : 0;
    for (int i = 0;; ++i) {
      const int buf = i & 1;
      if (i >= 2) mbar_wait(&slot_empty[buf], ((i >> 1) - 1) & 1);
      const int w = __shfl_sync(0xffffffffu, w_next, 0);
      WorkItem* si = &s_item[buf];
      if (w >= P.n_units) {
        if (lane == 0) si->valid = 0;
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&ent_full[buf]);
          mbar_arrive(&item_full[buf]);
        }
        break;
      }
      if (lane == 0) w_next = atomicAdd(P.work_counter, 1);
      if (lane < kItemInts) reinterpret_cast<int*>(si)[lane] = reinterpret_cast<const int*>(P.units + w)[lane];
      __syncwarp();
      const int n_ent = si->n_entries, n_mem = si->n_mem, kvh = si->kvh;
      const int64_t eoff = si->entry_off;
      PageRef* se = s_ent0 + buf * kMaxEntries;
      uint32_t* rag = reinterpret_cast<uint32_t*>(smem + kOffRag) + buf * 4;
      if (lane < 4) rag[lane] = 0u;
      __syncwarp();
      for (int j = lane; j < n_ent; j += 32) {
        const PageRef ref = P.arena[eoff + j];
        se[j] = ref.page >= 0 ? ref : make_ref(0, 0, 0);  // an unset entry reads no token (never expected)
        // a block with a page that is not 16 full slots from slot 0 (or past the unit's end) needs slot masks
        if (ref.page < 0 || ref_begin(ref) != 0 || ref_count(ref) != kPageTokens || ((j + 1 == n_ent) && (n_ent & 3)))
          atomicOr(&rag[(j >> 2) >> 5], 1u << ((j >> 2) & 31));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ent_full[buf]);  // the TMA lanes may stream this unit's pages
      const uint32_t half_bytes = (uint32_t)P.R * 128;
      if (i == 0) pdl_wait();  // the Q tile of this launch is complete and visible
      if (i >= 1) mbar_wait(q_free, (i - 1) & 1);  // the previous unit's Q tile is in TMEM
      const int copies = si->copies, rpc = 128 / copies;
      if (lane == 0) mbar_arrive_expect_tx(&item_full[buf], (uint32_t)kNH * half_bytes * (uint32_t)(n_mem * copies));
      __syncwarp();
      if (lane < kNH * n_mem * copies) {  // (member, half, copy): n_mem * R * copies <= 128 rows
        const int m = (lane / kNH) % n_mem, h = lane % kNH, cp = (lane / kNH) / n_mem;
        const int b = si->members[m];
        uint8_t* dst = smem + kOffQ + h * kQHalf + (cp * rpc) * 128 + m * half_bytes;
        const __nv_bfloat16* src = P.q_tile + (((size_t)b * P.kv_heads + kvh) * kNH + h) * (size_t)P.R * 64;
        bulk_g2s(dst, src, half_bytes, &item_full[buf]);
      }
    }
  } else if (warp == kWarpTma) {
    // ---------------- TMA: keeps the K and V rings full across work units ----------------
    // K and V streams (lanes 0-7 K, 8-15 V).  K slots free after Q.K^T, V slots after P.V.
    if (lane < 4 * kTmaLanesPerBlkGroup * 2) {
      // kTmaGroups 4-lane groups per stream; group j copies block g + j of every kTmaGroups-block
      // step.  A block whose 4 page ids are consecutive is 16 KiB of contiguous HBM in the
      // head-major plane (common.cuh) and goes as ONE bulk copy; otherwise lane p copies page p
      // (tools/microbench/mb_gather.cu: random 4 KiB copies need several issuing lanes to approach
      // the HBM bandwidth, 16 KiB copies reach it from one)
      constexpr int kTmaGroups = kTmaLanesPerBlkGroup;
      const size_t head_stride = (size_t)P.num_pages * kPageTokens * HD;
      const bool is_k = lane < 4 * kTmaGroups;
      const int sl_lane = lane % (4 * kTmaGroups);
      const int sub = sl_lane & 3, grp = sl_lane >> 2;
      const unsigned gmask = 0xFu << (lane & ~3);  // this lane's 4-lane group
      const int nsl = is_k ? kKSlots : kVSlots;
      uint64_t* fb = is_k ? kfull : vfull;
      uint64_t* eb = is_k ? kempty : vempty;
      uint8_t* rb = is_k ? ring : smem + kOffVRing;
      const __nv_bfloat16* plane = is_k ? P.kplane : P.vplane;
      int g0 = 0;  // first block of the unit (global block counter)
      for (int i = 0;; ++i) {
        const int buf = i & 1;
        mbar_wait(&ent_full[buf], (i >> 1) & 1);
        const WorkItem* si = &s_item[buf];
        if (!si->valid) break;
        const int n_ent = si->n_entries;
        const int nblk = (n_ent + kBlkPages - 1) / kBlkPages;
        const __nv_bfloat16* hplane = plane + (size_t)si->kvh * head_stride;
        const PageRef* se = s_ent0 + buf * kMaxEntries;
        for (int blk = grp; blk < nblk; blk += kTmaGroups) {
          const int g = g0 + blk;
          const int e0 = blk * kBlkPages;
          const int sl = g % nsl, np = min(kBlkPages, n_ent - e0);
          if (g >= nsl) mbar_wait(&eb[sl], ((g / nsl) - 1) & 1);
          uint8_t* dst = rb + sl * kSlotBytes;
          const int pg = sub < np ? se[e0 + sub].page : -1;
          const int p0 = __shfl_sync(gmask, pg, lane & ~3);
          const bool run = __all_sync(gmask, np == kBlkPages && pg == p0 + sub);
          if (sub == 0) mbar_arrive_expect_tx(&fb[sl], (uint32_t)np * kPB);
          __syncwarp(gmask);  // the expected bytes are registered before any copy can complete
          if (run) {
            if (sub == 0) bulk_g2s(dst, hplane + (size_t)p0 * (kPageTokens * HD), kRunBytes, &fb[sl]);
          } else if (sub < np) {
            bulk_g2s(dst + sub * kPB, hplane + (size_t)pg * (kPageTokens * HD), kPB, &fb[sl]);
          }
        }
        g0 += nblk;
        // every lane of the stream is done with the unit's entries before the slot is released
        __syncwarp(is_k ? (0xFFFFFFFFu >> (32 - 4 * kTmaGroups)) : ((0xFFFFFFFFu >> (32 - 4 * kTmaGroups)) << (4 * kTmaGroups)));
        if (sl_lane == 0) mbar_arrive(&slot_empty[buf]);  // this stream no longer reads the unit's entries
      }
    }
  } else if (warp == kWarpQk) {
    // ---------------- QK issuer: Q -> TMEM per unit, S_g = Q . K_g^T per block ----------------
    // Both issuers run converged with one elected lane issuing (prefill_tc3.cu: warp-uniform
    // descriptors stay in uniform registers, no per-MMA waterfall on an SMSP shared with softmax warps).
    const uint64_t qdesc0 = tc::sw128_desc(smem_u32(smem + kOffQ), 16, 1024);
    const uint64_t kdesc0 = tc::sw128_desc(smem_u32(ring), 16, 16 * HD);  // 8-token groups 16 * HD bytes apart
    int g = 0;
    for (int i = 0;; ++i) {
      const int ub = i & 1;
      mbar_wait(&item_full[ub], (i >> 1) & 1);
      const WorkItem* si = &s_item[ub];
      const int valid = si->valid, n_ent = si->n_entries;
      if (!valid) break;
      const int nblk = (n_ent + kBlkPages - 1) / kBlkPages;
      tc::fence_after();
      // the unit's Q tile smem -> TMEM (ordered after the previous unit's QK MMAs)
      if (tc::elect_one()) {
        issue_q_copy<HD>(qdesc0);
        tc::mma_commit(q_free);
      }
      __syncwarp();
      for (int blk = 0; blk < nblk; ++blk, ++g) {
        const int sb = g % kSBufs, sl = g % kKSlots;
        if (g >= kSBufs) mbar_wait(&pv_done[sb], ((g - kSBufs) / kSBufs) & 1);  // P(g - kSBufs) consumed
        mbar_wait(&kfull[sl], (g / kKSlots) & 1);
        tc::fence_after();
        const uint64_t kd = kdesc0 + (uint64_t)(sl * (kSlotBytes >> 4));
        if (tc::elect_one()) {
          switch (sb) {
            case 0: issue_qk_mmas<0, HD>(kd); break;
            case 1: issue_qk_mmas<1, HD>(kd); break;
            case 2: issue_qk_mmas<2, HD>(kd); break;
            case 3: issue_qk_mmas<3, HD>(kd); break;
            default: issue_qk_mmas<4, HD>(kd); break;
          }
          tc::mma_commit(&s_full[sb]);
          tc::mma_commit(&kempty[sl]);
        }
        __syncwarp();
      }
      if (tc::elect_one()) tc::mma_commit(&slot_empty[ub]);  // Q smem tile consumed
      __syncwarp();
    }
  } else if (warp == kWarpPv) {
    // ---------------- PV issuer: O_par += P_g . V_g per block ----------------
    const uint64_t vdesc0 = tc::sw128_desc(smem_u32(smem + kOffVRing), 1024, 16 * HD);
    int g = 0;
    for (int i = 0;; ++i) {
      const int ub = i & 1;
      mbar_wait(&item_full[ub], (i >> 1) & 1);
      const WorkItem* si = &s_item[ub];
      const int valid = si->valid, n_ent = si->n_entries, copies = si->copies;
      __syncwarp();
      if (lane == 0) mbar_arrive(&slot_empty[ub]);  // header read
      if (!valid) break;
      const int nblk = (n_ent + kBlkPages - 1) / kBlkPages;
      for (int blk = 0; blk < nblk; ++blk, ++g) {
        const int sb = g % kSBufs;
        mbar_wait(&p_full[sb], (g / kSBufs) & 1);
        if (blk == 0 && i >= 2) mbar_wait(&o_empty[i & 1], ((i >> 1) - 1) & 1);  // epilogue drained O[i & 1]
        mbar_wait(&vfull[g % kVSlots], (g / kVSlots) & 1);
        tc::fence_after();
        const uint64_t vd = vdesc0 + (uint64_t)((g % kVSlots) * (kSlotBytes >> 4));
        const int np = n_ent - blk * kBlkPages;
        const uint32_t acc0 = blk > 0 ? 1u : 0u;  // the unit's first block opens O
        const uint32_t ocol = kColO + (uint32_t)(i & 1) * 128u;
        if (tc::elect_one()) {
          switch (sb) {
            case 0: issue_pv_mmas<0, HD>(vd, np, acc0, copies, ocol); break;
            case 1: issue_pv_mmas<1, HD>(vd, np, acc0, copies, ocol); break;
            case 2: issue_pv_mmas<2, HD>(vd, np, acc0, copies, ocol); break;
            case 3: issue_pv_mmas<3, HD>(vd, np, acc0, copies, ocol); break;
            default: issue_pv_mmas<4, HD>(vd, np, acc0, copies, ocol); break;
          }
          tc::mma_commit(&vempty[g % kVSlots]);  // also certifies PV(g) to the softmax (O rescale)
          tc::mma_commit(&pv_done[sb]);
          if (blk == nblk - 1) tc::mma_commit(&o_full[i & 1]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ---------------- softmax: 8 warps, one block at a time (softmax_unit) ----------------
    const int q = warp & 3, half = (warp - 4) >> 2;
    const int r = q * 32 + lane;
    float* xmax = reinterpret_cast<float*>(smem + kOffFlag);
    int g = 0;
    for (int i = 0;; ++i) {
      const int buf = i & 1;
      mbar_wait(&item_full[buf], (i >> 1) & 1);
      const WorkItem* si = &s_item[buf];
      if (!si->valid) {
        if (i >= 2) mbar_wait(&o_empty[i & 1], ((i >> 1) - 1) & 1);
        if (warp == 4 && lane == 0) s_ep[i & 1].valid = 0;
        __syncwarp();
        if (lane == 0) mbar_arrive(&stat_full[i & 1]);
        break;
      }
      const int n_ent = si->n_entries, n_mem = si->n_mem, copies = si->copies;
      const PageRef* se = s_ent0 + buf * kMaxEntries;
      const uint32_t* rag = reinterpret_cast<const uint32_t*>(smem + kOffRag) + buf * 4;
      float m_ref, l;
      if (copies == 2)
        softmax_unit<2, HD>(P, g, n_ent, n_mem, se, rag, warp, lane, tmem, s_full, p_full, vempty, xmax, m_ref, l, i & 1);
      else
        softmax_unit<1, HD>(P, g, n_ent, n_mem, se, rag, warp, lane, tmem, s_full, p_full, vempty, xmax, m_ref, l, i & 1);
      // hand (m, l_half) and the unit header to the epilogue, release the unit slot
      // unit i - 2's epilogue read the stats / header slot of this parity
      if (i >= 2) mbar_wait(&o_empty[i & 1], ((i >> 1) - 1) & 1);
      s_stat[(i & 1) * 256 + half * 128 + r] = make_float2(m_ref, l);
      if (warp == 4 && lane < kItemInts) reinterpret_cast<int*>(s_ep + (i & 1))[lane] = reinterpret_cast<const int*>(si)[lane];
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&stat_full[i & 1]);
        mbar_arrive(&slot_empty[buf]);
      }
    }
  } else if (warp >= 12) {
    // ---------------- epilogue warpgroup: sum row copies, output or split-KV partial ----------------
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    float* xch = reinterpret_cast<float*>(smem + kOffXch);  // [copy - 1][row in copy][16]
    for (int i = 0;; ++i) {
      const int par = i & 1;
      mbar_wait(&stat_full[par], (i >> 1) & 1);
      const WorkItem* ep = s_ep + par;
      const float2* st2 = s_stat + par * 256;
      if (!ep->valid) break;
      const int n_mem = ep->n_mem, kvh = ep->kvh, F = ep->copies;
      const int qpc = 4 / F, rpc = 32 * qpc;
      const int c = q / qpc, lq = q % qpc, lr = r - c * rpc;
      const int mi = lr / P.R, hl = lr % P.R;
      const bool warp_active = lq * 32 < n_mem * P.R;
      const bool active = c == 0 && mi < n_mem && hl < P.gqa;
      const int b = active ? ep->members[mi] : 0;
      const int64_t slot = ep->slot_base + mi;
      // every copy and warp half shares the reference; the row's mass is the sum of the parts
      float2 ml = make_float2(st2[lr].x, 0.f);
      for (int cc = 0; cc < F; ++cc) ml.y += st2[cc * rpc + lr].y + st2[128 + cc * rpc + lr].y;
      mbar_wait(&o_full[par], (i >> 1) & 1);
      const uint32_t ocol = lane_base + kColO + par * 128;
      tc::fence_after();
      const int head = kvh * P.gqa + hl;
      const int nslots = active ? P.slot_cnt[b] : 0;
      const int64_t orow = (int64_t)b * P.q_heads + head;
      const float inv = ml.y > 0.f ? 1.f / ml.y : 0.f;
      if (F == 1) {
#pragma unroll 1
        for (int k = 0; k < HD / 32; ++k) {  // 32-column chunks of O
          float o[32];
          if (warp_active) {
            tc::tmem_ld32(ocol + k * 32, o);
            tc::tmem_wait_ld();
          }
          if (active) {
            if (nslots == 1) {
              store_row<HD>(P, orow, k, o, inv);
            } else {
              float4* dst = reinterpret_cast<float4*>(P.part_o + (slot * P.q_heads + head) * HD + k * 32);
#pragma unroll
              for (int e = 0; e < 8; ++e) __stcg(dst + e, make_float4(o[4 * e], o[4 * e + 1], o[4 * e + 2], o[4 * e + 3]));
            }
          }
        }
      } else {
#pragma unroll 1
        for (int k = 0; k < HD / 16; ++k) {  // 16-column chunks of O
          float o[16];
          if (warp_active) {
            tc::tmem_ldN<16>(ocol + k * 16, o);
            tc::tmem_wait_ld();
          }
          if (F > 1) {
            if (c > 0 && warp_active)
  #pragma unroll
              for (int e = 0; e < 16; e += 4)
                *reinterpret_cast<float4*>(&xch[((c - 1) * rpc + lr) * 16 + e]) = make_float4(o[e], o[e + 1], o[e + 2], o[e + 3]);
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (c == 0 && warp_active)
              for (int cc = 1; cc < F; ++cc)
  #pragma unroll
                for (int e = 0; e < 16; e += 4) {
                  const float4 x = *reinterpret_cast<const float4*>(&xch[((cc - 1) * rpc + lr) * 16 + e]);
                  o[e] += x.x;
                  o[e + 1] += x.y;
                  o[e + 2] += x.z;
                  o[e + 3] += x.w;
                }
            asm volatile("bar.sync 1, 128;" ::: "memory");
          }
          if (active) {
            if (nslots == 1) {
              store_row16<HD>(P, orow, k, o, inv);
            } else {
              float4* dst = reinterpret_cast<float4*>(P.part_o + (slot * P.q_heads + head) * HD + k * 16);
  #pragma unroll
              for (int e = 0; e < 4; ++e) __stcg(dst + e, make_float4(o[4 * e], o[4 * e + 1], o[4 * e + 2], o[4 * e + 3]));
            }
          }
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[par]);
      if (active && nslots > 1) __stcg(P.part_ml + slot * P.q_heads + head, ml);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(P.work_counter + 1, 1) == (int)gridDim.x - 1) {
    P.work_counter[0] = 0;  // every CTA has stopped claiming: re-arm the queue for the next launch
    P.work_counter[1] = 0;
  }
  if (warp == kWarpQk) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, kTmemCols);
  }
}

// Split-KV combine for handles with more than one partial slot: one warp per (handle, q head),
// float4 per lane, log-sum-exp over the handle's slots (single-slot handles were written by the
// decode epilogue directly).
constexpr int kCombineWarps = 4;       // narrow mode: pairs per CTA
constexpr int kCombineWideWarps = 16;
constexpr int kMultiRec = 10;          // ints per multi-slot handle: b, slot count, up to 8 slots (narrow mode)  // wide mode: warps merging one pair's slots (a 135K context has 68+ slots)
// Split-KV combine.  wide = 1: one CTA per (handle, q head), warp w merges slots w, w + 4, ...
// online (log-sum-exp), two slots' loads in flight, then warp 0 merges the four partial states
// (a long single context has one slot per chunk: 132 at the 135K-token C5 context).  wide = 0
// (every handle has few slots, e.g. C2's prefix + private chunk): one warp per (handle, q head).
__global__ void __launch_bounds__(32 * kCombineWideWarps) combine_kernel(
    const float* __restrict__ part_o, const float2* __restrict__ part_ml, const int32_t* __restrict__ multi,
    int n_multi, const int32_t* __restrict__ slot_ptr, const int32_t* __restrict__ slot_idx, int q_heads,
    void* __restrict__ out, int out_f32, int wide, int hd) {
  pdl_wait();  // programmatic launch behind decode_tc_kernel: its partials are visible after this
  pdl_launch_dependents();  // the next step's append may start its launch
  __shared__ float s_m[kCombineWideWarps], s_l[kCombineWideWarps];
  __shared__ float4 s_acc[kCombineWideWarps][32];
  const int nwarps = (int)(blockDim.x >> 5);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = wide ? blockIdx.x : blockIdx.x * kCombineWarps + warp;
  if (pair >= n_multi * q_heads) return;  // narrow mode only (warp-uniform)
  const int h = pair % q_heads;
  const bool dims = lane * 4 < hd;  // float4 of dims per lane (lanes 16-31 idle at head dim 64)
  // multi: per handle {b, slot count, its <= 8 slots} (kMultiRec ints), so the narrow path needs one load
  // before the partials' (instead of multi -> slot_ptr -> slot_idx -> partials)
  const int rv = lane < kMultiRec ? __ldg(multi + (size_t)(pair / q_heads) * kMultiRec + lane) : 0;
  const int b = __shfl_sync(0xffffffffu, rv, 0);
  if (!wide) {
    const int ns = __shfl_sync(0xffffffffu, rv, 1);
    float2 ml[kMultiRec - 2];
    float4 v[kMultiRec - 2];
#pragma unroll
    for (int u = 0; u < kMultiRec - 2; ++u) {
      const int64_t sl = __shfl_sync(0xffffffffu, rv, 2 + u);
      ml[u] = make_float2(-INFINITY, 0.f);
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (u < ns) {
        ml[u] = part_ml[sl * q_heads + h];
        if (dims) v[u] = *reinterpret_cast<const float4*>(&part_o[(sl * q_heads + h) * hd + lane * 4]);
      }
    }
    float m = -INFINITY;
#pragma unroll
    for (int u = 0; u < kMultiRec - 2; ++u) m = fmaxf(m, ml[u].x);
    float l = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < kMultiRec - 2; ++u)
      if (ml[u].x != -INFINITY) {
        const float w = fast_exp2(ml[u].x - m);
        l += w * ml[u].y;
        acc = make_float4(acc.x + w * v[u].x, acc.y + w * v[u].y, acc.z + w * v[u].z, acc.w + w * v[u].w);
      }
    if (!dims) return;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const int64_t at = ((int64_t)b * q_heads + h) * hd + lane * 4;
    if (out_f32) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + at) =
          make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    } else {
      uint2 pk;
      pk.x = pack_bf16(acc.x * inv, acc.y * inv);
      pk.y = pack_bf16(acc.z * inv, acc.w * inv);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + at) = pk;
    }
    return;
  }
  const int s0 = slot_ptr[b], s1 = slot_ptr[b + 1];
  const int first = wide ? s0 + warp : s0, step = wide ? nwarps : 1;
  float m = -INFINITY, l = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  auto merge = [&](float2 ml, float4 v) {
    if (ml.x == -INFINITY) return;
    const float nm = fmaxf(m, ml.x);
    const float a = m == -INFINITY ? 0.f : fast_exp2(m - nm), w = fast_exp2(ml.x - nm);
    acc = make_float4(acc.x * a + w * v.x, acc.y * a + w * v.y, acc.z * a + w * v.z, acc.w * a + w * v.w);
    l = l * a + w * ml.y;
    m = nm;
  };
  for (int s = first; s < s1; s += 2 * step) {
    const int64_t sa = slot_idx[s];
    const bool two = s + step < s1;
    const int64_t sb = two ? slot_idx[s + step] : sa;
    const float2 mla = part_ml[sa * q_heads + h], mlb = part_ml[sb * q_heads + h];
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 va = dims ? *reinterpret_cast<const float4*>(&part_o[(sa * q_heads + h) * hd + lane * 4]) : z4;
    const float4 vb = dims ? *reinterpret_cast<const float4*>(&part_o[(sb * q_heads + h) * hd + lane * 4]) : z4;
    merge(mla, va);
    if (two) merge(mlb, vb);
  }
  if (wide) {
    if (lane == 0) {
      s_m[warp] = m;
      s_l[warp] = l;
    }
    s_acc[warp][lane] = acc;
    __syncthreads();
    if (warp != 0) return;
    m = -INFINITY;
    l = 0.f;
    acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int w = 0; w < nwarps; ++w) merge(make_float2(s_m[w], s_l[w]), s_acc[w][lane]);
  }
  const float inv = l > 0.f ? 1.f / l : 0.f;
  const int64_t at = ((int64_t)b * q_heads + h) * hd + lane * 4;
  if (!dims) return;
  if (out_f32) {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + at) =
        make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  } else {
    uint2 pk;
    pk.x = pack_bf16(acc.x * inv, acc.y * inv);
    pk.y = pack_bf16(acc.z * inv, acc.w * inv);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + at) = pk;
  }
}

// RoPE pre-pass: rotates every query once (toy_model.cpp:30-41 at the handle's position) and
// writes it as the decode kernel's Q operand tile [n][kv_heads][hd / 64 halves][R rows][64 dims],
// SWIZZLE_128B (chunk c of row hl at c ^ (hl & 7)); rows hl >= gqa are zero.  One thread per
// 16-byte chunk.
__global__ void rope_q_tile_kernel(const __nv_bfloat16* __restrict__ q, const int32_t* __restrict__ pos, int n,
                                   int kv_heads, int gqa, int R, const RopeTable rt, __nv_bfloat16* __restrict__ tile) {
  // launched PDL-dependent on the append: wait for it (and, transitively, everything before it)
  // BEFORE releasing decode_tc, whose TMA lanes read the page tables and KV planes ahead of their
  // own griddepcontrol.wait
  pdl_wait();
  pdl_launch_dependents();  // decode_tc may start its prologue (every CTA of this grid is running)
  __shared__ double s_inv[kMaxHeadDim / 2];
  const double* inv = rope_stage(rt, s_inv);
  const int hd = rt.hd, lg = hd == 128 ? 4 : 3;  // log2 16-byte chunks per row
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = ((int64_t)n * kv_heads * R) << lg;
  if (x >= total) return;
  const int c = (int)(x & ((1 << lg) - 1));  // 16-byte chunk of the hd-dim row
  const int hl = (int)((x >> lg) % R);
  const int64_t bk = (x >> lg) / R;          // b * kv_heads + kvh
  const int b = (int)(bk / kv_heads), kvh = (int)(bk % kv_heads);
  uint4 v = make_uint4(0, 0, 0, 0);
  if (hl < gqa) {
    const int head = kvh * gqa + hl;
    v = *reinterpret_cast<const uint4*>(q + ((int64_t)b * kv_heads * gqa + head) * hd + c * 8);
    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&v);
    const int p = pos[b];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float cs, sn;
      rope_cs(p, inv[c * 4 + j], cs, sn);
      const float2 ab = __bfloat1622float2(h2[j]);
      h2[j] = __floats2bfloat162_rn(ab.x * cs - ab.y * sn, ab.x * sn + ab.y * cs);
    }
  }
  const int half = c >> 3, cc = c & 7;
  const int64_t dst = ((bk * (hd >> 6) + half) * R + hl) * 64 + ((cc ^ (hl & 7)) << 3);
  *reinterpret_cast<uint4*>(tile + dst) = v;
}

}  // namespace

struct DecodePlanCache {
  std::vector<uint64_t> handles;
  std::vector<int64_t> sig;  // per handle: n_entries, lineage size
  int q_heads = 0;
  // host plan
  std::vector<WorkItem> units;
  std::vector<int32_t> slot_ptr, slot_idx, slot_cnt, multi;  // multi: handles with > 1 slot
  std::vector<int32_t> multi_rec;  // per multi handle: b, slot count, its first 8 slots (combine_kernel)
  std::vector<int32_t> tail_item, tail_c0;  // per handle: item holding its private tail chunk (-1 none)
  int32_t n_slots = 0;
  mv_decode_plan_info info{};
  // device copies
  WorkItem* d_units = nullptr;
  int32_t *d_slot_ptr = nullptr, *d_slot_idx = nullptr, *d_slot_cnt = nullptr, *d_multi = nullptr;
  __nv_bfloat16* d_q_tile = nullptr;
  float* d_part_o = nullptr;
  float2* d_part_ml = nullptr;
  size_t cap_units = 0, cap_q = 0, cap_ptr = 0, cap_idx = 0, cap_cnt = 0, cap_multi = 0, cap_slots = 0;
  bool smem_set = false;
  int num_sms = 148;
  int* d_counter = nullptr;
  // optional kernel timing (mv_attn_decode_kernel_timing): an event pair around decode_tc per call
  std::vector<cudaEvent_t> t_begin, t_end;
  int t_used = 0;
  // pinned double-buffered staging for in-place plan updates (no implicit stream sync)
  WorkItem* h_stage[2] = {nullptr, nullptr};
  size_t cap_stage = 0;
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  int stage_k = 0;
  ~DecodePlanCache() {
    for (int k = 0; k < 2; ++k) {
      if (h_stage[k]) cudaFreeHost(h_stage[k]);
      if (stage_ev[k]) cudaEventDestroy(stage_ev[k]);
    }
    cudaFree(d_counter);
    for (auto e : t_begin) cudaEventDestroy(e);
    for (auto e : t_end) cudaEventDestroy(e);
    cudaFree(d_units);
    cudaFree(d_q_tile);
    cudaFree(d_slot_ptr);
    cudaFree(d_slot_idx);
    cudaFree(d_slot_cnt);
    cudaFree(d_multi);
    cudaFree(d_part_o);
    cudaFree(d_part_ml);
  }
};

void destroy_plan(DecodePlanCache* p) { delete p; }

template <typename T>
static mv_status ensure_dev(T*& p, size_t& cap, size_t n) {
  if (n <= cap) return MV_OK;
  cudaFree(p);
  p = nullptr;
  size_t c = std::max<size_t>(2 * n, cap * 2);  // headroom: re-plans of growing tables rarely reallocate
  MV_CUDA_TRY(cudaMalloc(&p, sizeof(T) * c));
  cap = c;
  return MV_OK;
}

static int rows_per_member(int gqa) {
  int R = 8;
  while (R < gqa) R *= 2;
  return R;
}

static void build_plan(PagedStore& st, DecodePlanCache& pc, const uint64_t* hs, int n, int kv_heads, int gqa,
                       int num_sms) {
  pc.units.clear();
  std::vector<std::vector<int32_t>> slots_of(n);
  int32_t n_slots = 0;
  int64_t unique_tokens = 0, naive_tokens = 0;
  const int R = rows_per_member(gqa);
  const int max_members = std::max(1, std::min(kMaxMem, 128 / R));

  // group id -> member batch indices (in batch order)
  std::unordered_map<uint64_t, std::vector<int32_t>> group_members;
  std::vector<HandleRec*> recs(n);
  for (int b = 0; b < n; ++b) {
    recs[b] = st.find(hs[b]);
    naive_tokens += recs[b]->n_tokens();
    for (auto& lg : recs[b]->lineage) group_members[lg.group].push_back(b);
  }

  // cascade units: (arena offset, entry range, members)
  struct Seg {
    int64_t off;
    int32_t e0, e1;
    std::vector<int32_t> mem;
    int32_t tail_of;  // handle whose private tail this segment is (-1: shared segment)
  };
  std::vector<Seg> segs;
  int64_t total_pages = 0;
  auto add_seg = [&](int64_t off, int32_t e0, int32_t e1, std::vector<int32_t> mem, int64_t tokens, int32_t tail_of) {
    if (e1 <= e0 || mem.empty()) return;
    unique_tokens += tokens;
    total_pages += e1 - e0;
    segs.push_back({off, e0, e1, std::move(mem), tail_of});
  };
  std::unordered_map<uint64_t, bool> done;
  for (int b = 0; b < n; ++b) {
    const HandleRec* r = recs[b];
    int32_t prev_e = 0;
    int64_t prev_t = 0;
    for (auto& lg : r->lineage) {
      auto& mem = group_members[lg.group];
      if (mem.size() >= 2 && !done[lg.group]) {
        done[lg.group] = true;
        add_seg(r->arena_off, prev_e, lg.entries, mem, lg.tokens - prev_t, -1);
      }
      if (mem.size() >= 2) {
        prev_e = lg.entries;
        prev_t = lg.tokens;
      }
    }
    // private remainder (single-holder lineage segments coalesce here)
    add_seg(r->arena_off, prev_e, r->n_entries(), std::vector<int32_t>{b}, r->n_tokens() - prev_t, b);
  }

  // split-KV chunk: the largest power of two <= 256 pages that still gives >= 1.5 waves of units
  // over the SMs.  Sweeps (with the parallel combine): C5's single 135K context 0.123 ms at 256
  // pages vs 0.138 at 64; C2 and C4 best at 128-256.  Fewer, longer units mean fewer partials.
  const int64_t target_units = (int64_t)num_sms * 3 / 2;
  int chunk = kMaxChunk;
  while (chunk > 16 && total_pages * kv_heads / chunk < target_units) chunk /= 2;

  std::vector<WorkItem> items;
  std::vector<int32_t> tags, tag_c0;  // per item: handle whose private tail it ends (-1), its first entry
  for (const Seg& s : segs) {
    const int32_t npg = s.e1 - s.e0;
    const int32_t nchunks = (npg + chunk - 1) / chunk;
    for (int32_t c = 0; c < nchunks; ++c) {
      const int32_t c0 = s.e0 + (int32_t)((int64_t)npg * c / nchunks);
      const int32_t c1 = s.e0 + (int32_t)((int64_t)npg * (c + 1) / nchunks);
      const int ngroups = (int)((s.mem.size() + max_members - 1) / max_members);
      for (int gi = 0; gi < ngroups; ++gi) {
        // balanced member groups
        const size_t m0 = s.mem.size() * gi / ngroups, m1 = s.mem.size() * (gi + 1) / ngroups;
        WorkItem w;
        std::memset(&w, 0, sizeof w);
        w.entry_off = s.off + c0;
        w.n_entries = c1 - c0;
        w.n_mem = (int32_t)(m1 - m0);
        w.slot_base = n_slots;
        w.valid = 1;
        const int rows = w.n_mem * R;
        // Wide cascade units (33-64 rows: two lane quadrants, so two SMSPs carry their softmax)
        // get a second row copy in the other two quadrants, each copy exponentiating half of
        // every block's columns: the softmax spreads over all four SMSPs (C2 +2%).
        w.copies = (rows > 32 && rows <= 64) ? 2 : 1;
        for (size_t k = m0; k < m1; ++k) {
          w.members[k - m0] = s.mem[k];
          slots_of[s.mem[k]].push_back(n_slots + (int32_t)(k - m0));
        }
        n_slots += w.n_mem;
        items.push_back(w);
        tags.push_back(s.tail_of >= 0 && c == nchunks - 1 ? s.tail_of : -1);
        tag_c0.push_back(c0);
      }
    }
  }
  auto longest_first = [&](std::vector<int32_t>& ord) {
    ord.resize(items.size());
    for (size_t k = 0; k < ord.size(); ++k) ord[k] = (int32_t)k;
    std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) {
      const WorkItem &a = items[x], &b = items[y];
      return a.n_entries != b.n_entries ? a.n_entries > b.n_entries : a.n_mem > b.n_mem;
    });
  };
  // Tail split: the dynamic queue ends with its smallest units, and when it runs dry every SM finishes
  // the unit it holds at a different time (C2 measured SMs idle ~10% of the launch).  The last two
  // waves of units are therefore halved (4-page-block aligned); a handle whose chunk is split gets one
  // more split-KV slot.
  {
    std::vector<int32_t> ord;
    longest_first(ord);
    std::vector<int32_t> split;
    int64_t acc = 0;
    for (size_t k = ord.size(); k-- > 0 && acc < 2 * (int64_t)num_sms;) {
      acc += kv_heads;
      if (items[ord[k]].n_entries >= 2 * kBlkPages) split.push_back(ord[k]);
    }
    for (int32_t it : split) {
      WorkItem a = items[it];
      const int32_t half = (a.n_entries / 2 + kBlkPages - 1) / kBlkPages * kBlkPages;
      WorkItem b = a;
      b.entry_off = a.entry_off + half;
      b.n_entries = a.n_entries - half;
      b.slot_base = n_slots;
      for (int m = 0; m < b.n_mem; ++m) slots_of[b.members[m]].push_back(n_slots + m);
      n_slots += b.n_mem;
      items[it].n_entries = half;
      items.push_back(b);
      tags.push_back(tags[it]);  // the second half ends where the chunk ended (a growing private tail)
      tag_c0.push_back(tag_c0[it] + half);
      tags[it] = -1;
    }
  }
  // longest-first (then widest-first) for the dynamic queue: the tail is made of the smallest units
  std::vector<int32_t> order(items.size());
  for (size_t k = 0; k < order.size(); ++k) order[k] = (int32_t)k;
  std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
    const WorkItem &a = items[x], &b = items[y];
    return a.n_entries != b.n_entries ? a.n_entries > b.n_entries : a.n_mem > b.n_mem;
  });
  pc.tail_item.assign(n, -1);
  pc.tail_c0.assign(n, 0);
  pc.units.reserve(items.size() * kv_heads);
  for (size_t k = 0; k < order.size(); ++k) {
    const int32_t it = order[k];
    if (tags[it] >= 0) {
      pc.tail_item[tags[it]] = (int32_t)k;
      pc.tail_c0[tags[it]] = tag_c0[it];
    }
    for (int h = 0; h < kv_heads; ++h) {
      WorkItem u = items[it];
      u.kvh = h;
      pc.units.push_back(u);
    }
  }

  pc.slot_ptr.assign(n + 1, 0);
  pc.slot_cnt.assign(n, 0);
  pc.slot_idx.clear();
  pc.multi.clear();
  for (int b = 0; b < n; ++b) {
    pc.slot_cnt[b] = (int32_t)slots_of[b].size();
    pc.slot_ptr[b + 1] = pc.slot_ptr[b] + pc.slot_cnt[b];
    if (pc.slot_cnt[b] > 1) pc.multi.push_back(b);
    pc.slot_idx.insert(pc.slot_idx.end(), slots_of[b].begin(), slots_of[b].end());
  }
  pc.n_slots = n_slots;
  pc.info.units = (int32_t)segs.size();
  pc.info.chunks = chunk;
  pc.info.work_items = (int32_t)items.size();
  pc.info.partial_slots = n_slots;
  pc.info.unique_kv_tokens = unique_tokens;
  pc.info.naive_kv_tokens = naive_tokens;
}

}  // namespace mv

using namespace mv;

extern "C" mv_status mv_attn_decode(mv_kv_store* s, int32_t layer, const uint64_t* hs, int32_t n, int32_t q_heads,
                                    const void* d_q, const int32_t* d_positions, void* d_out, int32_t out_dtype) {
  if (!s || !s->impl) return fail(MV_ERR_INVALID_ARGUMENT, "null store");
  PagedStore& st = *s->impl;
  const mv_kv_config& cfg = st.cfg();
  if (cfg.kv_heads <= 0 || layer < 0 || layer >= cfg.layers)
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_attn_decode: no attention plane for this layer");
  if (n <= 0) return n == 0 ? MV_OK : fail(MV_ERR_INVALID_ARGUMENT, "mv_attn_decode: n < 0");
  if (q_heads <= 0 || q_heads % cfg.kv_heads) return fail(MV_ERR_INVALID_ARGUMENT, "q_heads % kv_heads != 0");
  const int gqa = q_heads / cfg.kv_heads;
  if (gqa > 128) return fail(MV_ERR_INVALID_ARGUMENT, "GQA group larger than 128 heads");
  if (!d_q || !d_positions || !d_out) return fail(MV_ERR_INVALID_ARGUMENT, "null buffer");
  if (out_dtype != 0 && out_dtype != 1) return fail(MV_ERR_INVALID_ARGUMENT, "out_dtype must be 0 (bf16) or 1 (fp32)");

  if (!st.plan) st.plan = new DecodePlanCache();
  DecodePlanCache& pc = *st.plan;
  if (!pc.smem_set) {
    MV_CUDA_TRY(cudaFuncSetAttribute(decode_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    MV_CUDA_TRY(cudaFuncSetAttribute(decode_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    int dev = 0;
    MV_CUDA_TRY(cudaGetDevice(&dev));
    MV_CUDA_TRY(cudaDeviceGetAttribute(&pc.num_sms, cudaDevAttrMultiProcessorCount, dev));
    MV_CUDA_TRY(cudaMalloc(&pc.d_counter, 2 * sizeof(int)));  // [0] work queue, [1] finished CTAs
    MV_CUDA_TRY(cudaMemset(pc.d_counter, 0, 2 * sizeof(int)));
    pc.smem_set = true;
  }
  // plan signature: the handle list plus each table's entry count and lineage depth
  std::vector<int64_t> sig(3 * (size_t)n);
  for (int b = 0; b < n; ++b) {
    HandleRec* r = st.find(hs[b]);
    if (!r) return fail(MV_ERR_DOUBLE_RELEASE, "handle " + std::to_string(hs[b]) + " is unknown or already released");
    if (r->n_tokens() == 0) return fail(MV_ERR_INVALID_ARGUMENT, "mv_attn_decode: empty context");
    sig[3 * b] = r->n_entries();
    sig[3 * b + 1] = (int64_t)r->lineage.size();
    sig[3 * b + 2] = r->arena_off;
  }
  const bool same_set = pc.q_heads == q_heads && pc.handles.size() == (size_t)n &&
                        std::equal(pc.handles.begin(), pc.handles.end(), hs) && pc.sig.size() == sig.size();
  bool same = same_set && pc.sig == sig;
  cudaStream_t stream = st.stream();
  if (same_set && !same) {
    // Decode appends grow only each branch's private tail: bump its tail chunk in place (one upload,
    // no re-plan) while the chunk fits; anything else (new lineage, moved table) re-plans.
    bool incr = true;
    for (int b = 0; b < n && incr; ++b) {
      if (sig[3 * b + 1] != pc.sig[3 * b + 1] || sig[3 * b + 2] != pc.sig[3 * b + 2] || sig[3 * b] < pc.sig[3 * b]) incr = false;
      else if (sig[3 * b] != pc.sig[3 * b] &&
               (pc.tail_item[b] < 0 || sig[3 * b] - pc.tail_c0[b] > std::min(kMaxEntries, pc.info.chunks + 16)))
        incr = false;  // a tail chunk may outgrow the plan's chunk size by 16 pages before a re-plan
    }
    if (incr) {
      for (int b = 0; b < n; ++b) {
        if (sig[3 * b] == pc.sig[3 * b]) continue;
        const int it = pc.tail_item[b];
        for (int h = 0; h < cfg.kv_heads; ++h) pc.units[(size_t)it * cfg.kv_heads + h].n_entries = (int32_t)(sig[3 * b] - pc.tail_c0[b]);
      }
      // pinned double-buffered staging: an async copy that does not drain the stream
      if (pc.cap_stage < pc.units.size()) {
        for (int k = 0; k < 2; ++k) {
          if (pc.h_stage[k]) cudaFreeHost(pc.h_stage[k]);
          pc.h_stage[k] = nullptr;
          MV_CUDA_TRY(cudaMallocHost(&pc.h_stage[k], sizeof(WorkItem) * pc.units.size()));
          if (!pc.stage_ev[k]) MV_CUDA_TRY(cudaEventCreateWithFlags(&pc.stage_ev[k], cudaEventDisableTiming));
        }
        pc.cap_stage = pc.units.size();
      }
      const int k = pc.stage_k;
      pc.stage_k ^= 1;
      MV_CUDA_TRY(cudaEventSynchronize(pc.stage_ev[k]));  // the copy that last used this buffer
      std::memcpy(pc.h_stage[k], pc.units.data(), sizeof(WorkItem) * pc.units.size());
      MV_CUDA_TRY(cudaMemcpyAsync(pc.d_units, pc.h_stage[k], sizeof(WorkItem) * pc.units.size(),
                                  cudaMemcpyHostToDevice, stream));
      MV_CUDA_TRY(cudaEventRecord(pc.stage_ev[k], stream));
      pc.sig = sig;
      same = true;
    }
  }
  if (!same) {
    build_plan(st, pc, hs, n, cfg.kv_heads, gqa, pc.num_sms);
    pc.handles.assign(hs, hs + n);
    pc.sig = sig;
    pc.q_heads = q_heads;
    if (mv_status e = ensure_dev(pc.d_units, pc.cap_units, pc.units.size())) return e;
    if (mv_status e = ensure_dev(pc.d_slot_ptr, pc.cap_ptr, pc.slot_ptr.size())) return e;
    if (mv_status e = ensure_dev(pc.d_slot_idx, pc.cap_idx, std::max<size_t>(1, pc.slot_idx.size()))) return e;
    if (mv_status e = ensure_dev(pc.d_slot_cnt, pc.cap_cnt, pc.slot_cnt.size())) return e;
    if (mv_status e = ensure_dev(pc.d_multi, pc.cap_multi, std::max<size_t>(1, pc.multi.size() * kMultiRec))) return e;
    if (!pc.multi.empty()) {
      pc.multi_rec.assign(pc.multi.size() * kMultiRec, 0);
      for (size_t k = 0; k < pc.multi.size(); ++k) {
        const int32_t b = pc.multi[k], ns = pc.slot_cnt[b];
        int32_t* rec = pc.multi_rec.data() + k * kMultiRec;
        rec[0] = b;
        rec[1] = ns;
        for (int j = 0; j < ns && j < kMultiRec - 2; ++j) rec[2 + j] = pc.slot_idx[pc.slot_ptr[b] + j];
      }
      MV_CUDA_TRY(cudaMemcpyAsync(pc.d_multi, pc.multi_rec.data(), sizeof(int32_t) * pc.multi_rec.size(),
                                  cudaMemcpyHostToDevice, stream));
    }
    const size_t old_slots = pc.cap_slots;
    // 2x headroom: later re-plans split growing tails into more chunks (more partial slots)
    if (mv_status e = ensure_dev(pc.d_part_ml, pc.cap_slots, std::max<size_t>(1, (size_t)pc.n_slots * q_heads * 2)))
      return e;
    if (pc.cap_slots != old_slots || !pc.d_part_o) {
      cudaFree(pc.d_part_o);
      pc.d_part_o = nullptr;
      MV_CUDA_TRY(cudaMalloc(&pc.d_part_o, sizeof(float) * pc.cap_slots * kMaxHeadDim));
    }
    MV_CUDA_TRY(cudaMemcpyAsync(pc.d_units, pc.units.data(), sizeof(WorkItem) * pc.units.size(),
                                cudaMemcpyHostToDevice, stream));
    MV_CUDA_TRY(cudaMemcpyAsync(pc.d_slot_ptr, pc.slot_ptr.data(), sizeof(int32_t) * pc.slot_ptr.size(),
                                cudaMemcpyHostToDevice, stream));
    MV_CUDA_TRY(cudaMemcpyAsync(pc.d_slot_idx, pc.slot_idx.data(), sizeof(int32_t) * pc.slot_idx.size(),
                                cudaMemcpyHostToDevice, stream));
    MV_CUDA_TRY(cudaMemcpyAsync(pc.d_slot_cnt, pc.slot_cnt.data(), sizeof(int32_t) * pc.slot_cnt.size(),
                                cudaMemcpyHostToDevice, stream));
    // pageable sources: each copy is staged before its call returns (it drains the stream, which is
    // acceptable for a full re-plan; in-place updates above use pinned staging)
  }
  const int R = rows_per_member(gqa);
  const int hd = cfg.head_dim;
  if (mv_status e = ensure_dev(pc.d_q_tile, pc.cap_q, (size_t)n * cfg.kv_heads * R * hd)) return e;
  {
    const int64_t chunks = (int64_t)n * cfg.kv_heads * R * (hd / 8);
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)((chunks + 255) / 256));
    lc.blockDim = dim3(256);
    lc.stream = stream;
    lc.attrs = pdl;
    lc.numAttrs = 1;
    MV_CUDA_TRY(cudaLaunchKernelEx(&lc, rope_q_tile_kernel, (const __nv_bfloat16*)d_q, d_positions, n,
                                   cfg.kv_heads, gqa, R, st.rope(), pc.d_q_tile));
    MV_LAUNCH_CHECK();
  }
  DecodeParams P;
  P.arena = st.d_arena;
  P.kplane = st.k_planes()[layer];
  P.vplane = st.v_planes()[layer];
  P.q_tile = pc.d_q_tile;
  P.units = pc.d_units;
  P.n_units = (int)pc.units.size();
  P.work_counter = pc.d_counter;
  P.part_o = pc.d_part_o;
  P.part_ml = pc.d_part_ml;
  P.slot_cnt = pc.d_slot_cnt;
  P.slot_ptr = pc.d_slot_ptr;
  P.slot_idx = pc.d_slot_idx;
  P.out = d_out;
  P.out_f32 = out_dtype == 1;
  P.kv_heads = cfg.kv_heads;
  P.num_pages = cfg.num_pages;
  P.q_heads = q_heads;
  P.gqa = gqa;
  P.R = R;
  P.scale_log2 = 1.4426950408889634f / sqrtf((float)hd);
  const int grid = std::min(P.n_units, pc.num_sms);
  // decode_tc and combine are launched programmatically dependent on the kernel before them
  // (PDL): their launch latency and prologue overlap the predecessor's tail
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(kThreads);
  lc.dynamicSmemBytes = kSmem;
  lc.stream = stream;
  lc.attrs = pdl;
  lc.numAttrs = 1;
  // kernel timing: the events sit between the RoPE pass and decode_tc (which then cannot overlap its
  // prologue with the RoPE pass), so this measures the whole decode_tc launch
  const bool timed = pc.t_used < (int)pc.t_begin.size();
  if (timed) MV_CUDA_TRY(cudaEventRecord(pc.t_begin[pc.t_used], stream));
  if (hd == 128) MV_CUDA_TRY(cudaLaunchKernelEx(&lc, decode_tc_kernel<128>, P));
  else MV_CUDA_TRY(cudaLaunchKernelEx(&lc, decode_tc_kernel<64>, P));
  if (timed) MV_CUDA_TRY(cudaEventRecord(pc.t_end[pc.t_used++], stream));
  MV_LAUNCH_CHECK();
  if (!pc.multi.empty()) {
    int max_slots = 0;
    for (int32_t b : pc.multi) max_slots = std::max(max_slots, pc.slot_cnt[b]);
    const int wide = max_slots > 8 ? 1 : 0;
    const size_t pairs = pc.multi.size() * (size_t)q_heads;
    lc.gridDim = dim3((unsigned)(wide ? pairs : (pairs + kCombineWarps - 1) / kCombineWarps));
    lc.blockDim = dim3(32 * (wide ? kCombineWideWarps : kCombineWarps));
    lc.dynamicSmemBytes = 0;
    MV_CUDA_TRY(cudaLaunchKernelEx(&lc, combine_kernel, (const float*)pc.d_part_o, (const float2*)pc.d_part_ml,
                                   (const int32_t*)pc.d_multi, (int)pc.multi.size(), (const int32_t*)pc.d_slot_ptr,
                                   (const int32_t*)pc.d_slot_idx, q_heads, d_out, (int)(out_dtype == 1), wide, hd));
    MV_LAUNCH_CHECK();
  }
  return MV_OK;
}

extern "C" mv_status mv_attn_decode_plan_info(mv_kv_store* s, mv_decode_plan_info* out) {
  if (!s || !s->impl || !out) return fail(MV_ERR_INVALID_ARGUMENT, "null argument");
  if (!s->impl->plan) {
    std::memset(out, 0, sizeof *out);
    return MV_OK;
  }
  *out = s->impl->plan->info;
  return MV_OK;
}

extern "C" mv_status mv_attn_decode_kernel_timing(mv_kv_store* s, int32_t max_calls, float* h_ms, int32_t* h_n) {
  if (!s || !s->impl) return fail(MV_ERR_INVALID_ARGUMENT, "null store");
  if (!s->impl->plan) s->impl->plan = new DecodePlanCache();
  DecodePlanCache& pc = *s->impl->plan;
  if (h_n) {  // read back the recorded calls (waits for the last one)
    const int n = pc.t_used;
    if (n > 0 && !h_ms) return fail(MV_ERR_INVALID_ARGUMENT, "mv_attn_decode_kernel_timing: null h_ms");
    for (int k = 0; k < n; ++k) {
      MV_CUDA_TRY(cudaEventSynchronize(pc.t_end[k]));
      MV_CUDA_TRY(cudaEventElapsedTime(h_ms + k, pc.t_begin[k], pc.t_end[k]));
    }
    *h_n = n;
  }
  if (max_calls < 0) return fail(MV_ERR_INVALID_ARGUMENT, "max_calls < 0");
  while ((int)pc.t_begin.size() < max_calls) {
    cudaEvent_t a, b;
    MV_CUDA_TRY(cudaEventCreate(&a));
    MV_CUDA_TRY(cudaEventCreate(&b));
    pc.t_begin.push_back(a);
    pc.t_end.push_back(b);
  }
  while ((int)pc.t_begin.size() > max_calls) {
    cudaEventDestroy(pc.t_begin.back());
    cudaEventDestroy(pc.t_end.back());
    pc.t_begin.pop_back();
    pc.t_end.pop_back();
  }
  pc.t_used = 0;
  return MV_OK;
}
