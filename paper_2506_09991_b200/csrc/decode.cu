// decode.cu — K4: branch-parallel paged decode attention (split-KV, cascade over fork lineage).
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
// Units are split into <= 64-page chunks (split-KV); a work item = (chunk, <= 8 handles).
//
// Kernel (one CTA per (work item, KV head)):
//   warp 6      : TMA warp — 1-D bulk copies (TMA engine) of each 4 KiB K and V page-head
//                 block into a 15-stage smem ring, mbarrier complete_tx signalling; it runs
//                 ahead across work-item boundaries (persistent kernel, dynamic item queue).
//   warp 7      : staging warp — claims the next (chunk, kv head) item and stages its page
//                 entries and RoPE-rotated Q rows into a double buffer.
//   warps 0..5  : 3 consumer pairs; pair p takes pages p, p+3, ...  Tokens are the MMA M
//                 dimension and query rows the N dimension (mma.sync m16n8k16, swapped
//                 operands), so 40 rows = 5 n8-tiles with no padding; S^T -> P^T goes
//                 register-to-register through movmatrix.  Both warps of a pair compute
//                 S = K.Q^T (Q lives in registers); each accumulates O^T for half of the
//                 128 head dims.  Online softmax in the log2 domain, fp32 accumulation.
//   epilogue    : the 3 pairs' (m, l, O) are merged through smem and written as one
//                 partial per (handle, q head); a combine kernel merges the partials of
//                 each handle's chunks (log-sum-exp) into bf16 outputs.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "store.hpp"

namespace mv {

namespace {

constexpr int kConsumerWarps = 6;
constexpr int kConsumerThreads = kConsumerWarps * 32;
constexpr int kDecThreads = kConsumerThreads + 64;  // + TMA warp + staging warp = 8 warps (255 regs)
constexpr int kStages = 15;
constexpr int kStageBytes = 2 * kPageTokens * kHeadDim * 2;  // K + V page-head blocks (8 KiB)
constexpr int kMaxNT = 5;                                   // <= 40 query rows per item
constexpr int kMaxRows = kMaxNT * 8;
constexpr int kChunkPages = 64;                             // split-KV chunk (pages)
constexpr float kLazyRescale = 8.f;                         // log2-domain headroom before O is rescaled
constexpr int kRowSlots = 144;                              // epilogue rows: 6 streams x 24 or 3 x 40
constexpr int kSmemRing = kStages * kStageBytes;            // 120 KiB
constexpr int kSmemQ = kMaxRows * kHeadDim * 2;             // 10 KiB per buffer
constexpr int kSmemEnt = kChunkPages * 8;                   // 512 B per buffer
constexpr int kSmemO = kRowSlots * kHeadDim * 4;            // 72 KiB epilogue
constexpr int kSmemML = kRowSlots * 2 * 4;
constexpr int kOffQ = kSmemRing;
constexpr int kOffEnt = kOffQ + 2 * kSmemQ;
constexpr int kOffO = kOffEnt + 2 * kSmemEnt;
constexpr int kOffML = kOffO + kSmemO;
constexpr int kOffItem = kOffML + kSmemML;
constexpr int kItemSlotBytes = 128;
constexpr int kOffBar = kOffItem + 2 * kItemSlotBytes;
constexpr int kOffTag = kOffBar + (2 * kStages + 4) * 8;
constexpr int kDecSmem = kOffTag + kStages * 4;

// Consumer split of an item with NT row tiles: NT <= 3 -> every warp owns all rows and its own
// page stream (6 streams); NT 4-5 -> warp pairs split the rows (ceil(NT/2) + floor(NT/2)) and
// share a page stream (3 streams). No warp repeats another's Q.K^T work.
__host__ __device__ constexpr int row_groups(int nt) { return nt <= 3 ? 1 : 2; }

constexpr int kMaxMembers = 8;  // handles per work item (8 x GQA 5 = 40 rows)

struct __align__(16) WorkItem {
  int64_t entry_off;             // absolute arena index of the chunk's first entry
  int32_t n_entries;
  int32_t n_mem;                 // handles (query groups) sharing this chunk
  int32_t slot_base;             // partial slot of the first member
  int32_t nt;                    // n8 row tiles (ceil(n_mem * gqa / 8))
  int32_t members[kMaxMembers];  // batch indices
  int32_t pad[2];
};
static_assert(sizeof(WorkItem) == 64, "WorkItem is one 64 B line");

struct ItemSlot {      // what the producer hands the consumers for one (item, kv head)
  WorkItem it;
  int32_t kvh;
  int32_t valid;
};

static_assert(sizeof(ItemSlot) <= kItemSlotBytes, "item slot overflows its smem reservation");

struct DecodeParams {
  const PageRef* arena;
  const __nv_bfloat16* kplane;
  const __nv_bfloat16* vplane;
  const __nv_bfloat16* q_rot; // [n][q_heads][128], RoPE already applied (rope_q_kernel)
  const WorkItem* items;
  float* part_o;              // [slots][q_heads][128]
  float2* part_ml;            // [slots][q_heads]
  int* work_counter;          // dynamic (item, kv head) scheduler
  int n_work;                 // items * kv_heads
  int kv_heads, q_heads, gqa;
  float scale_log2;           // log2(e) / sqrt(128)
  int diag;                   // diagnostics: 1 = skip math (pipeline only), 2 = skip loads (math only)
  unsigned long long* trace;  // optional per-item timeline (MV_DECODE_TRACE)
  RopeTable rope;
};

// Consumer side of one work item for one warp: rows [nt0*8, (nt0+NTW)*8), pages
// j = stream, stream + n_streams, ... . S^T = K.Q^T (tokens are the MMA M dimension), online
// softmax in the log2 domain with lazy rescaling, P^T via movmatrix, O^T += V^T.P^T over all
// 128 head dims (8 m-tiles).
template <int NTW>
__device__ __forceinline__ void consume_rows(const DecodeParams& P, const WorkItem& it, int gbase, int stream,
                                             int n_streams, int nt0, uint8_t* ring, const uint8_t* sq,
                                             const PageRef* s_ent, uint64_t* full, uint64_t* empty,
                                             int empty_count, float* s_ml, float* s_o, const int* s_tag) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;

  uint32_t qb[NTW][8][2];
  const uint32_t sq_base = smem_u32(sq);
#pragma unroll
  for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      int row = (nt0 + nt) * 8 + (lane & 7);
      int chunk = ks * 2 + ((lane >> 3) & 1);
      // Q rows land in smem by bulk copy (unswizzled); 4-way conflicts once per item only
      ldmatrix_x2(qb[nt][ks][0], qb[nt][ks][1], sq_base + row * 256 + (chunk << 4));
    }

  float o[8][NTW][4];
#pragma unroll
  for (int mt = 0; mt < 8; ++mt)
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
      for (int k = 0; k < 4; ++k) o[mt][nt][k] = 0.f;
  float m_ref[NTW][2], l_run[NTW][2];
#pragma unroll
  for (int nt = 0; nt < NTW; ++nt) {
    m_ref[nt][0] = m_ref[nt][1] = -INFINITY;
    l_run[nt][0] = l_run[nt][1] = 0.f;
  }

  const int npages = it.n_entries;
  for (int j = stream; j < npages; j += n_streams) {
    const int gp = gbase + j;
    const int stage = gp % kStages;
    const PageRef ref = s_ent[j];
    const int vb = ref_begin(ref), ve = vb + ref_count(ref);
    // Streams consume stages out of order, so a stream may reach page gp while the stage still
    // holds page gp - kStages in flight; a bare parity wait would then match the previous phase.
    // The TMA warp tags the stage with gp before issuing it, which pins the phase.
    while (ld_volatile_s32(&s_tag[stage]) != gp) {
    }
    mbar_wait(&full[stage], (gp / kStages) & 1);
    if (P.diag == 1) {
      __syncwarp();
      if (lane == 0) mbar_arrive_n(&empty[stage], empty_count);
      continue;
    }
    const uint32_t kbase = smem_u32(ring + stage * kStageBytes);
    const uint32_t vbase = kbase + kPageTokens * kHeadDim * 2;

    float s[NTW][4];
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      uint32_t a[4];
      const int mi = lane >> 3;
      const int row = (mi & 1) * 8 + (lane & 7);
      const int chunk = ks * 2 + (mi >> 1);
      ldmatrix_x4(a[0], a[1], a[2], a[3], kbase + row * 256 + (swz_chunk(row, chunk) << 4));
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt) mma_bf16_16816(s[nt], a, qb[nt][ks][0], qb[nt][ks][1]);
    }

    const bool v0 = g >= vb && g < ve, v1 = g + 8 >= vb && g + 8 < ve;
    float x[NTW][4], mx[NTW][2];
    bool need = false;
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt) {
      x[nt][0] = v0 ? s[nt][0] * P.scale_log2 : -INFINITY;
      x[nt][1] = v0 ? s[nt][1] * P.scale_log2 : -INFINITY;
      x[nt][2] = v1 ? s[nt][2] * P.scale_log2 : -INFINITY;
      x[nt][3] = v1 ? s[nt][3] * P.scale_log2 : -INFINITY;
      mx[nt][0] = fmaxf(x[nt][0], x[nt][2]);
      mx[nt][1] = fmaxf(x[nt][1], x[nt][3]);
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        mx[nt][0] = fmaxf(mx[nt][0], __shfl_xor_sync(0xffffffffu, mx[nt][0], off));
        mx[nt][1] = fmaxf(mx[nt][1], __shfl_xor_sync(0xffffffffu, mx[nt][1], off));
      }
      need |= mx[nt][0] > m_ref[nt][0] + kLazyRescale || mx[nt][1] > m_ref[nt][1] + kLazyRescale;
    }
    if (__any_sync(0xffffffffu, need)) {
      // move the reference max (rare after the first pages): rescale l and O
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const float mn = fmaxf(m_ref[nt][c], mx[nt][c]);
          const float al = mn == -INFINITY ? 1.f : fast_exp2(m_ref[nt][c] - mn);
          m_ref[nt][c] = mn;
          l_run[nt][c] *= al;
#pragma unroll
          for (int mt = 0; mt < 8; ++mt) {
            o[mt][nt][c] *= al;
            o[mt][nt][2 + c] *= al;
          }
        }
    }
    uint32_t pb[NTW][2];
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt) {
      const float mu0 = m_ref[nt][0] == -INFINITY ? 0.f : m_ref[nt][0];
      const float mu1 = m_ref[nt][1] == -INFINITY ? 0.f : m_ref[nt][1];
      const float p0 = fast_exp2(x[nt][0] - mu0), p1 = fast_exp2(x[nt][1] - mu1);
      const float p2 = fast_exp2(x[nt][2] - mu0), p3 = fast_exp2(x[nt][3] - mu1);
      l_run[nt][0] += p0 + p2;
      l_run[nt][1] += p1 + p3;
      pb[nt][0] = movmatrix_trans(pack_bf16(p0, p1));
      pb[nt][1] = movmatrix_trans(pack_bf16(p2, p3));
    }

    // O^T (128 dims x rows) += V^T . P^T
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      uint32_t a[4];
      const int mi = lane >> 3;
      const int tok = (mi >> 1) * 8 + (lane & 7);
      const int chunk = mt * 2 + (mi & 1);
      ldmatrix_x4_trans(a[0], a[1], a[2], a[3], vbase + tok * 256 + (swz_chunk(tok, chunk) << 4));
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt) mma_bf16_16816(o[mt][nt], a, pb[nt][0], pb[nt][1]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_n(&empty[stage], empty_count);
  }

  // finish l (sum over the 8 token lanes g) and publish this stream's (m, l, O) rows
#pragma unroll
  for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float l = l_run[nt][c];
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
      l_run[nt][c] = l;
    }
  const int rows = it.nt * 8;
  asm volatile("bar.sync 1, %0;" ::"r"(kConsumerThreads));  // previous item's merge readers are done
  if (g == 0) {
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int r = (nt0 + nt) * 8 + 2 * t4 + c;
        s_ml[(stream * rows + r) * 2 + 0] = m_ref[nt][c];
        s_ml[(stream * rows + r) * 2 + 1] = l_run[nt][c];
      }
  }
#pragma unroll
  for (int mt = 0; mt < 8; ++mt)
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int dim = mt * 16 + g + (k >> 1) * 8;
        const int r = (nt0 + nt) * 8 + 2 * t4 + (k & 1);
        s_o[(stream * rows + r) * kHeadDim + dim] = o[mt][nt][k];
      }
}

// All consumer warps: merge the streams' partials and write one partial per (member, q head).
__device__ __forceinline__ void merge_streams(const DecodeParams& P, const ItemSlot& is, int n_streams,
                                              const float* s_ml, const float* s_o) {
  asm volatile("bar.sync 1, %0;" ::"r"(kConsumerThreads));
  const WorkItem& it = is.it;
  const int rows = it.nt * 8;
  const int nrows = it.n_mem * P.gqa;
  for (int x = threadIdx.x; x < nrows * (kHeadDim / 4); x += kConsumerThreads) {
    const int r = x / (kHeadDim / 4), d4 = (x % (kHeadDim / 4)) * 4;
    float m = -INFINITY;
    for (int st = 0; st < n_streams; ++st) m = fmaxf(m, s_ml[(st * rows + r) * 2]);
    const float mu = m == -INFINITY ? 0.f : m;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float l = 0.f;
    for (int st = 0; st < n_streams; ++st) {
      const float w = fast_exp2(s_ml[(st * rows + r) * 2] - mu);
      const float4 v = *reinterpret_cast<const float4*>(&s_o[(st * rows + r) * kHeadDim + d4]);
      acc.x += w * v.x;
      acc.y += w * v.y;
      acc.z += w * v.z;
      acc.w += w * v.w;
      l += w * s_ml[(st * rows + r) * 2 + 1];
    }
    const int mi = r / P.gqa, hl = r % P.gqa;
    const int64_t slot = it.slot_base + mi;
    const int head = is.kvh * P.gqa + hl;
    *reinterpret_cast<float4*>(&P.part_o[(slot * P.q_heads + head) * kHeadDim + d4]) = acc;
    if (d4 == 0) P.part_ml[slot * P.q_heads + head] = make_float2(m, l);
  }
}

// Persistent kernel: one CTA per SM pulls (chunk, kv head) work items from a global counter.
// The producer warp stages item i+1 (entries, rotated Q) and keeps the page ring full while
// the consumers finish item i, so per-item prologue/epilogue latency stays off the HBM path.
__global__ void __launch_bounds__(kDecThreads, 1) decode_kernel(DecodeParams P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  ItemSlot* s_item = reinterpret_cast<ItemSlot*>(smem + kOffItem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* empty = full + kStages;
  uint64_t* item_full = empty + kStages;
  uint64_t* item_empty = item_full + 2;
  float* s_o = reinterpret_cast<float*>(smem + kOffO);
  float* s_ml = reinterpret_cast<float*>(smem + kOffML);
  int* s_tag = reinterpret_cast<int*>(smem + kOffTag);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int st = threadIdx.x; st < kStages; st += blockDim.x) s_tag[st] = -1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&item_full[b], 32);
      mbar_init(&item_empty[b], kConsumerWarps + kStages);  // consumer warps + TMA lanes
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps + 1) {
    // ---------------- staging warp: claims work and stages entries + Q rows ----------------
    // Critical path per item is ~2 memory round trips: the next claim is issued one item
    // ahead, Q rows (pre-rotated) arrive by bulk copy on the item barrier itself.
    int w_next = lane == 0 ? atomicAdd(P.work_counter, 1) : 0;
    for (int iter = 0;; ++iter) {
      const int buf = iter & 1;
      if (iter >= 2) mbar_wait(&item_empty[buf], ((iter >> 1) - 1) & 1);
      const int w = __shfl_sync(0xffffffffu, w_next, 0);
      ItemSlot* is = &s_item[buf];
      if (w >= P.n_work) {
        if (lane == 0) is->valid = 0;
        __syncwarp();
        mbar_arrive(&item_full[buf]);
        break;
      }
      if (lane == 0) w_next = atomicAdd(P.work_counter, 1);
      const WorkItem it = P.items[w / P.kv_heads];
      const int kvh = w % P.kv_heads;
      uint8_t* sq = smem + kOffQ + buf * kSmemQ;
      const int qbytes = P.gqa * kHeadDim * 2;  // one handle's GQA group of q heads, contiguous
      if (lane == 0) {
        is->it = it;
        is->kvh = kvh;
        is->valid = 1;
        mbar_arrive_expect_tx(&item_full[buf], it.n_mem * qbytes);
      }
      __syncwarp();
      if (lane < it.n_mem) {
        const int b = it.members[lane];
        bulk_g2s(sq + lane * qbytes, P.q_rot + ((size_t)b * P.q_heads + kvh * P.gqa) * kHeadDim, qbytes,
                 &item_full[buf]);
      }
      PageRef* s_ent = reinterpret_cast<PageRef*>(smem + kOffEnt + buf * kSmemEnt);
      for (int j = lane; j < it.n_entries; j += 32) s_ent[j] = P.arena[it.entry_off + j];
      // zero the padding rows of the last n8 tile
      const int nrows = it.n_mem * P.gqa, rows = it.nt * 8;
      for (int x = lane; x < (rows - nrows) * 16; x += 32)
        *reinterpret_cast<uint4*>(sq + nrows * 256 + x * 16) = make_uint4(0, 0, 0, 0);
      __syncwarp();
      if (lane != 0) mbar_arrive(&item_full[buf]);  // lane 0 arrived with expect_tx
    }
    return;
  }

  if (warp == kConsumerWarps) {
    // ---------------- TMA warp: keeps the page ring full across item boundaries ----------------
    // Lane l (< kStages) owns ring stage l and issues every page that maps to it. One issuing
    // thread per stage matters: a single issuing thread serialises on its empty-barrier waits and
    // caps a CTA at ~15 GB/s (tools/microbench/mb_tma.cu: 2.3 TB/s vs 7.0 TB/s chip-wide).
    if (lane < kStages) {
      int gbase = 0;
      for (int iter = 0;; ++iter) {
        const int buf = iter & 1;
        mbar_wait(&item_full[buf], (iter >> 1) & 1);
        const ItemSlot* is = &s_item[buf];
        if (!is->valid) break;
        const PageRef* s_ent = reinterpret_cast<const PageRef*>(smem + kOffEnt + buf * kSmemEnt);
        const size_t head_off = (size_t)is->kvh * kPageTokens * kHeadDim;
        const int n_entries = is->it.n_entries;
        const size_t page_stride = (size_t)P.kv_heads * kPageTokens * kHeadDim;
        for (int j = ((lane - gbase) % kStages + kStages) % kStages; j < n_entries; j += kStages) {
          const int gp = gbase + j;
          if (gp >= kStages) mbar_wait(&empty[lane], ((gp / kStages) - 1) & 1);
          st_volatile_s32(&s_tag[lane], gp);
          uint8_t* dst = ring + lane * kStageBytes;
          if (P.diag == 2) {
            mbar_arrive(&full[lane]);
            continue;
          }
          const size_t src = (size_t)s_ent[j].page * page_stride + head_off;
          mbar_arrive_expect_tx(&full[lane], kStageBytes);
          bulk_g2s(dst, P.kplane + src, kStageBytes / 2, &full[lane]);
          bulk_g2s(dst + kStageBytes / 2, P.vplane + src, kStageBytes / 2, &full[lane]);
        }
        mbar_arrive(&item_empty[buf]);  // this lane no longer reads the item's entry list
        gbase += n_entries;
      }
    }
    return;
  }

  // ---------------- consumer warps ----------------
  int gbase = 0;
  unsigned long long* tr = P.trace ? P.trace + (size_t)blockIdx.x * 64 * 4 : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = globaltimer();
  for (int iter = 0;; ++iter) {
    const int buf = iter & 1;
    mbar_wait(&item_full[buf], (iter >> 1) & 1);
    const ItemSlot is = s_item[buf];
    if (tr && threadIdx.x == 0 && iter < 62) { tr[4 + iter * 4] = globaltimer(); tr[5 + iter * 4] = is.it.n_entries | ((unsigned long long)is.it.nt << 32); }
    if (!is.valid) break;
    const uint8_t* sq = smem + kOffQ + buf * kSmemQ;
    const PageRef* s_ent = reinterpret_cast<const PageRef*>(smem + kOffEnt + buf * kSmemEnt);
    const int nt = is.it.nt;
    const int G = row_groups(nt);
    const int n_streams = kConsumerWarps / G;
    const int stream = warp / G, half = warp % G;
    const int nta = (nt + 1) / 2;
    const int nt0 = G == 1 ? 0 : (half ? nta : 0);
    const int ntw = G == 1 ? nt : (half ? nt - nta : nta);
    // each stage is released by 2 arrivals: both warps of a pair, or one warp arriving twice
    const int ecount = G == 1 ? 2 : 1;
    switch (ntw) {
      case 1: consume_rows<1>(P, is.it, gbase, stream, n_streams, nt0, ring, sq, s_ent, full, empty, ecount, s_ml, s_o, s_tag); break;
      case 2: consume_rows<2>(P, is.it, gbase, stream, n_streams, nt0, ring, sq, s_ent, full, empty, ecount, s_ml, s_o, s_tag); break;
      default: consume_rows<3>(P, is.it, gbase, stream, n_streams, nt0, ring, sq, s_ent, full, empty, ecount, s_ml, s_o, s_tag); break;
    }
    // Q buffer and entry list of this item are no longer read: hand them back to the stager.
    __syncwarp();
    if (lane == 0) mbar_arrive(&item_empty[buf]);
    if (tr && threadIdx.x == 0 && iter < 62) tr[6 + iter * 4] = globaltimer();
    merge_streams(P, is, n_streams, s_ml, s_o);
    if (tr && threadIdx.x == 0 && iter < 62) tr[7 + iter * 4] = globaltimer();
    gbase += is.it.n_entries;
  }
}

// RoPE pre-pass: rotate every query once (toy_model.cpp:30-41 at the handle's position) so the
// decode kernel can bulk-copy Q rows; thread 0 also resets the work-item counter.
__global__ void rope_q_kernel(const __nv_bfloat16* __restrict__ q, const int32_t* __restrict__ pos, int n,
                              int q_heads, const RopeTable rt, __nv_bfloat16* __restrict__ q_rot, int* counter) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // one 16 B chunk (4 pairs)
  if (x == 0) *counter = 0;
  if (x >= (int64_t)n * q_heads * 16) return;
  const int c = (int)(x & 15);
  const int b = (int)(x / (16 * q_heads));
  uint4 v = *reinterpret_cast<const uint4*>(q + x * 8);
  __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&v);
  const int p = pos[b];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float cs, sn;
    rope_cs(p, rt.inv[c * 4 + j], cs, sn);
    const float2 ab = __bfloat1622float2(h2[j]);
    h2[j] = __floats2bfloat162_rn(ab.x * cs - ab.y * sn, ab.x * sn + ab.y * cs);
  }
  *reinterpret_cast<uint4*>(q_rot + x * 8) = v;
}

// Merge every handle's partials (log-sum-exp) into the output; one warp per (handle, q head),
// float4 per lane, single pass with online rescaling.
__global__ void combine_kernel(const float* __restrict__ part_o, const float2* __restrict__ part_ml,
                               const int32_t* __restrict__ slot_ptr, const int32_t* __restrict__ slot_idx, int n,
                               int q_heads, void* __restrict__ out, int out_f32) {
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= n * q_heads) return;
  const int b = wid / q_heads, h = wid % q_heads;
  const int s0 = slot_ptr[b], s1 = slot_ptr[b + 1];
  float m = -INFINITY, l = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s = s0; s < s1; ++s) {
    const int64_t sl = slot_idx[s];
    const float2 ml = part_ml[sl * q_heads + h];
    const float4 v = *reinterpret_cast<const float4*>(&part_o[(sl * q_heads + h) * kHeadDim + lane * 4]);
    const float mn = fmaxf(m, ml.x);
    if (mn == -INFINITY) continue;
    const float a = fast_exp2(m - mn), w = fast_exp2(ml.x - mn);
    acc.x = acc.x * a + w * v.x;
    acc.y = acc.y * a + w * v.y;
    acc.z = acc.z * a + w * v.z;
    acc.w = acc.w * a + w * v.w;
    l = l * a + w * ml.y;
    m = mn;
  }
  const float inv = l > 0.f ? 1.f / l : 0.f;
  const int64_t at = ((int64_t)b * q_heads + h) * kHeadDim + lane * 4;
  if (out_f32) {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + at) =
        make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  } else {
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
    __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&lo);
    pk.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + at) = pk;
  }
}

}  // namespace

struct DecodePlanCache {
  std::vector<uint64_t> handles;
  std::vector<int64_t> sig;  // per handle: n_entries, lineage size
  int q_heads = 0;
  // host plan
  std::vector<WorkItem> items;
  std::vector<int32_t> slot_ptr, slot_idx;
  int32_t n_slots = 0;
  mv_decode_plan_info info{};
  // device copies
  WorkItem* d_items = nullptr;
  int32_t *d_slot_ptr = nullptr, *d_slot_idx = nullptr;
  __nv_bfloat16* d_q_rot = nullptr;
  float* d_part_o = nullptr;
  float2* d_part_ml = nullptr;
  size_t cap_items = 0, cap_q_rot = 0, cap_ptr = 0, cap_idx = 0, cap_slots = 0;
  bool smem_set = false;
  int num_sms = 148;
  int* d_counter = nullptr;
  unsigned long long* d_trace = nullptr;
  ~DecodePlanCache() {
    cudaFree(d_counter);
    cudaFree(d_trace);
    cudaFree(d_items);
    cudaFree(d_q_rot);
    cudaFree(d_slot_ptr);
    cudaFree(d_slot_idx);
    cudaFree(d_part_o);
    cudaFree(d_part_ml);
  }
};

template <typename T>
static mv_status ensure_dev(T*& p, size_t& cap, size_t n) {
  if (n <= cap) return MV_OK;
  cudaFree(p);
  p = nullptr;
  size_t c = std::max<size_t>(n, cap * 2);
  MV_CUDA_TRY(cudaMalloc(&p, sizeof(T) * c));
  cap = c;
  return MV_OK;
}

static void build_plan(PagedStore& st, DecodePlanCache& pc, const uint64_t* hs, int n, int q_heads, int gqa) {
  pc.items.clear();
  std::vector<std::vector<int32_t>> slots_of(n);
  int32_t n_slots = 0;
  int64_t unique_tokens = 0, naive_tokens = 0;
  const int max_members = std::max(1, std::min(kMaxMembers, (kMaxNT * 8) / gqa));

  // group id -> member batch indices (in batch order)
  std::unordered_map<uint64_t, std::vector<int32_t>> group_members;
  std::vector<HandleRec*> recs(n);
  for (int b = 0; b < n; ++b) {
    recs[b] = st.find(hs[b]);
    naive_tokens += recs[b]->n_tokens();
    for (auto& lg : recs[b]->lineage) group_members[lg.group].push_back(b);
  }

  auto emit_unit = [&](int64_t src_off, int32_t e0, int32_t e1, const std::vector<int32_t>& mem, int64_t tokens) {
    if (e1 <= e0 || mem.empty()) return;
    unique_tokens += tokens;
    const int32_t npg = e1 - e0;
    const int32_t nchunks = (npg + kChunkPages - 1) / kChunkPages;
    for (int32_t c = 0; c < nchunks; ++c) {
      const int32_t c0 = e0 + (int32_t)((int64_t)npg * c / nchunks);
      const int32_t c1 = e0 + (int32_t)((int64_t)npg * (c + 1) / nchunks);
      for (size_t m0 = 0; m0 < mem.size(); m0 += max_members) {
        const int32_t nm = (int32_t)std::min<size_t>(max_members, mem.size() - m0);
        WorkItem w;
        std::memset(&w, 0, sizeof w);
        w.entry_off = src_off + c0;
        w.n_entries = c1 - c0;
        w.n_mem = nm;
        w.slot_base = n_slots;
        w.nt = (nm * gqa + 7) / 8;
        for (int32_t k = 0; k < nm; ++k) {
          w.members[k] = mem[m0 + k];
          slots_of[mem[m0 + k]].push_back(n_slots + k);
        }
        n_slots += nm;
        pc.items.push_back(w);
      }
    }
  };

  // shared cascade units: one per lineage group with >= 2 decoding holders
  std::unordered_map<uint64_t, bool> done;
  for (int b = 0; b < n; ++b) {
    const HandleRec* r = recs[b];
    int32_t prev_e = 0;
    int64_t prev_t = 0;
    for (auto& lg : r->lineage) {
      auto& mem = group_members[lg.group];
      if (mem.size() >= 2 && !done[lg.group]) {
        done[lg.group] = true;
        emit_unit(r->arena_off, prev_e, lg.entries, mem, lg.tokens - prev_t);
      }
      if (mem.size() >= 2) {
        prev_e = lg.entries;
        prev_t = lg.tokens;
      }
    }
    // private remainder (single-holder lineage segments coalesce here)
    emit_unit(r->arena_off, prev_e, r->n_entries(), std::vector<int32_t>{b}, r->n_tokens() - prev_t);
  }

  pc.slot_ptr.assign(n + 1, 0);
  pc.slot_idx.clear();
  for (int b = 0; b < n; ++b) {
    pc.slot_ptr[b + 1] = pc.slot_ptr[b] + (int32_t)slots_of[b].size();
    pc.slot_idx.insert(pc.slot_idx.end(), slots_of[b].begin(), slots_of[b].end());
  }
  pc.n_slots = n_slots;
  pc.info.units = 0;
  pc.info.chunks = 0;
  pc.info.work_items = (int32_t)pc.items.size();
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
  if (gqa > kMaxNT * 8) return fail(MV_ERR_INVALID_ARGUMENT, "GQA group larger than 40 heads");
  if (!d_q || !d_positions || !d_out) return fail(MV_ERR_INVALID_ARGUMENT, "null buffer");
  if (out_dtype != 0 && out_dtype != 1) return fail(MV_ERR_INVALID_ARGUMENT, "out_dtype must be 0 (bf16) or 1 (fp32)");

  if (!st.plan) st.plan = new DecodePlanCache();
  DecodePlanCache& pc = *st.plan;
  // plan signature: the handle list plus each table's entry count and lineage depth
  std::vector<int64_t> sig(2 * (size_t)n);
  for (int b = 0; b < n; ++b) {
    HandleRec* r = st.find(hs[b]);
    if (!r) return fail(MV_ERR_DOUBLE_RELEASE, "handle " + std::to_string(hs[b]) + " is unknown or already released");
    if (r->n_tokens() == 0) return fail(MV_ERR_INVALID_ARGUMENT, "mv_attn_decode: empty context");
    sig[2 * b] = r->n_entries();
    sig[2 * b + 1] = (int64_t)r->lineage.size();
  }
  const bool same = pc.q_heads == q_heads && pc.handles.size() == (size_t)n &&
                    std::equal(pc.handles.begin(), pc.handles.end(), hs) && pc.sig == sig;
  cudaStream_t stream = st.stream();
  if (!same) {
    build_plan(st, pc, hs, n, q_heads, gqa);
    pc.handles.assign(hs, hs + n);
    pc.sig = sig;
    pc.q_heads = q_heads;
    if (mv_status e = ensure_dev(pc.d_items, pc.cap_items, pc.items.size())) return e;
    if (mv_status e = ensure_dev(pc.d_slot_ptr, pc.cap_ptr, pc.slot_ptr.size())) return e;
    if (mv_status e = ensure_dev(pc.d_slot_idx, pc.cap_idx, std::max<size_t>(1, pc.slot_idx.size()))) return e;
    size_t old_slots = pc.cap_slots;
    if (mv_status e = ensure_dev(pc.d_part_ml, pc.cap_slots, (size_t)pc.n_slots * q_heads)) return e;
    if (pc.cap_slots != old_slots || !pc.d_part_o) {
      cudaFree(pc.d_part_o);
      MV_CUDA_TRY(cudaMalloc(&pc.d_part_o, sizeof(float) * pc.cap_slots * kHeadDim));
    }
    MV_CUDA_TRY(cudaMemcpyAsync(pc.d_items, pc.items.data(), sizeof(WorkItem) * pc.items.size(),
                                cudaMemcpyHostToDevice, stream));
    MV_CUDA_TRY(cudaMemcpyAsync(pc.d_slot_ptr, pc.slot_ptr.data(), sizeof(int32_t) * pc.slot_ptr.size(),
                                cudaMemcpyHostToDevice, stream));
    MV_CUDA_TRY(cudaMemcpyAsync(pc.d_slot_idx, pc.slot_idx.data(), sizeof(int32_t) * pc.slot_idx.size(),
                                cudaMemcpyHostToDevice, stream));
  }
  if (!pc.smem_set) {
    MV_CUDA_TRY(cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDecSmem));
    int dev = 0;
    MV_CUDA_TRY(cudaGetDevice(&dev));
    MV_CUDA_TRY(cudaDeviceGetAttribute(&pc.num_sms, cudaDevAttrMultiProcessorCount, dev));
    MV_CUDA_TRY(cudaMalloc(&pc.d_counter, sizeof(int)));
    pc.smem_set = true;
  }
  DecodeParams P;
  P.arena = st.d_arena;
  P.kplane = st.k_planes()[layer];
  P.vplane = st.v_planes()[layer];
  if (mv_status e = ensure_dev(pc.d_q_rot, pc.cap_q_rot, (size_t)n * q_heads * kHeadDim)) return e;
  P.q_rot = pc.d_q_rot;
  P.items = pc.d_items;
  P.part_o = pc.d_part_o;
  P.part_ml = pc.d_part_ml;
  P.kv_heads = cfg.kv_heads;
  P.q_heads = q_heads;
  P.gqa = gqa;
  P.scale_log2 = 1.4426950408889634f / sqrtf((float)kHeadDim);
  P.rope = st.rope();
  {
    const char* dg = getenv("MV_DECODE_DIAG");
    P.diag = dg ? atoi(dg) : 0;
    P.trace = nullptr;
    if (getenv("MV_DECODE_TRACE")) {
      if (!pc.d_trace) MV_CUDA_TRY(cudaMalloc(&pc.d_trace, sizeof(unsigned long long) * 148 * 64 * 4 * 2));
      MV_CUDA_TRY(cudaMemsetAsync(pc.d_trace, 0, sizeof(unsigned long long) * 148 * 64 * 4 * 2, stream));
      P.trace = pc.d_trace;
    }
  }
  {
    const int64_t chunks = (int64_t)n * q_heads * 16;
    rope_q_kernel<<<(unsigned)((chunks + 255) / 256), 256, 0, stream>>>(
        (const __nv_bfloat16*)d_q, d_positions, n, q_heads, st.rope(), pc.d_q_rot, pc.d_counter);
    MV_LAUNCH_CHECK();
  }
  P.work_counter = pc.d_counter;
  P.n_work = (int)pc.items.size() * cfg.kv_heads;
  const int grid = std::min(P.n_work, pc.num_sms);
  decode_kernel<<<grid, kDecThreads, kDecSmem, stream>>>(P);
  MV_LAUNCH_CHECK();
  if (P.trace) {
    std::vector<unsigned long long> h(148 * 64 * 4);
    MV_CUDA_TRY(cudaMemcpyAsync(h.data(), pc.d_trace, h.size() * 8, cudaMemcpyDeviceToHost, stream));
    MV_CUDA_TRY(cudaStreamSynchronize(stream));
    if (FILE* f = fopen(getenv("MV_DECODE_TRACE"), "wb")) {
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
  const int warps = n * q_heads;
  combine_kernel<<<(warps + 7) / 8, 256, 0, stream>>>(pc.d_part_o, pc.d_part_ml, pc.d_slot_ptr, pc.d_slot_idx, n,
                                                      q_heads, d_out, out_dtype == 1);
  MV_LAUNCH_CHECK();
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
