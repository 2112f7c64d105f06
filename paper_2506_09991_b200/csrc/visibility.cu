// visibility.cu — K1: tag stream -> Multiverse positions, segment ids and per-token exclusion
// intervals (the compact form of the structured mask), plus the dense-mask and prefill
// tile-map expansions.
//
// Reference behaviour replaced:
//   grammar.cpp:156-294  Parser (error kinds and their precedence)
//   dag.cpp:117-187      DagBuilder::visit_block (segments, visibility parents)
//   dag.cpp:203-222      assign_positions: segment start = 1 + max(parent end), root 0
//   dag.cpp:227-263      visibility_sets + build_mask
//
// Algorithm (phases 1-2: one CTA per sequence streaming through it in tiles; phase 3: one CTA
// per 1024-token tile):
//   1. parallel: compact the indices of tag tokens (ids 0..9) with a block scan; every
//      token also records the rank of the last tag at or before it, and its segment id from a
//      second scan over segment-start flags.
//   2. one thread walks only the tags (a few per block, not per token) with the grammar
//      automaton, validating structure exactly in the reference parser's order and
//      computing, per tag, its position (sibling <Path>s restart at plan_end+1,
//      <Conclusion> at max_path_end+1) and the exclusion-interval node that applies from
//      that tag on: inside path q >= 2 of block B, rows [first <Path> of B, <Path>_q)
//      are invisible (sibling paths never see each other). Interval nodes form a
//      persistent stack (one node per <Path>_q, q >= 2), so nesting costs O(1) per tag.
//   3. parallel (visibility_fill_kernel): each token takes pos = pos(last tag) + distance and
//      copies its <= D intervals from the node chain.  The walker reads its tags and node
//      depths from shared memory.  C3 (16K tokens): 59 us (was 144 us as one CTA).
#include <algorithm>

#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace mv {
namespace {

constexpr int kVisThreads = 512;
constexpr int kVisItems = 8;                      // tokens per thread per tile
constexpr int kVisTile = kVisThreads * kVisItems;  // 4096
constexpr int kMaxFrames = 256;                   // open <Parallel> nesting handled by the walker
constexpr int kMaxIntervals = 64;                 // exclusion intervals per token the mask consumers accept
constexpr int kSmemTags = 4096;                   // tags (and interval nodes) the walker reads from smem

struct SeqWs {
  int32_t* tag_idx;   // [n] sequence-local index of the k-th tag
  int32_t* tag_pos;   // [n] position of the k-th tag token
  int32_t* tag_node;  // [n] interval node applying from the k-th tag on (-1 none)
  int32_t* last_tag;  // [n] rank of the last tag at or before token i (-1 none)
  int4* nodes;        // [n] interval nodes {lo, hi, parent, depth}
  int32_t* single;    // [n] per <Conclusion> tag rank: 1 if its block has exactly one path
};

__device__ inline SeqWs seq_ws(void* ws, int64_t off, int64_t n) {
  // Each sequence owns a contiguous workspace slice of 12*n int32 (a multiple of 4 int32 per token keeps
  // the int4 node array 16-byte aligned for every sequence offset).
  int32_t* base = reinterpret_cast<int32_t*>(ws) + off * 12;
  SeqWs w;
  w.tag_idx = base;
  w.tag_pos = base + n;
  w.tag_node = base + 2 * n;
  w.last_tag = base + 3 * n;
  w.nodes = reinterpret_cast<int4*>(base + 4 * n);
  w.single = base + 8 * n;
  return w;
}

enum Phase : int32_t {
  kAfterParOpen = 0,  // expect <Goal>; text here is a stray gap (grammar.cpp:181)
  kGoalPreamble,      // free text allowed (take_text, grammar.cpp:183)
  kInOutline,         // outline body
  kAfterOutline,      // gap: <Outline> or </Goal>
  kAfterGoal,         // gap: <Path> expected
  kInPath,            // path body: text, nested <Parallel>, </Path>
  kAfterPath,         // gap: <Path> or <Conclusion>
  kInConclusion,      // conclusion text
  kAfterConclusion,   // gap: </Parallel>
};

struct Frame {
  int32_t phase, outlines, paths;
  int32_t plan_end, max_path_end;
  int32_t first_path_idx;
  int32_t enclosing_node;  // interval node of the context the block sits in
};

__global__ void __launch_bounds__(kVisThreads) visibility_kernel(const int32_t* __restrict__ tokens,
                                                                  const int64_t* __restrict__ offsets, int max_depth,
                                                                  int32_t* __restrict__ positions,
                                                                  int32_t* __restrict__ seg_id,
                                                                  int32_t* __restrict__ excl,
                                                                  int32_t* __restrict__ status, void* ws) {
  using Scan = cub::BlockScan<int, kVisThreads>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ int s_carry, s_seg_carry;
  __shared__ Frame frames[kMaxFrames];
  __shared__ int s_ntags;
  __shared__ int s_err;
  // the single-thread walk is latency-bound: its per-tag inputs (tag index, tag kind) and the
  // interval-node depths it chains through live in shared memory for the first kSmemTags tags
  __shared__ int s_tag_idx[kSmemTags];
  __shared__ int8_t s_tag_kind[kSmemTags];
  __shared__ int s_node_w[kSmemTags];

  const int s = blockIdx.x;
  const int64_t off = offsets[s];
  const int n = (int)(offsets[s + 1] - off);
  const int32_t* tok = tokens + off;
  SeqWs w = seq_ws(ws, off, n);

  // ---- phase 1: tag compaction + last-tag rank, segment ids ----
  if (threadIdx.x == 0) {
    s_carry = 0;
    s_seg_carry = 0;
  }
  __syncthreads();
  for (int base = 0; base < n; base += kVisTile) {
    int flag[kVisItems], rank[kVisItems], sflag[kVisItems], sid[kVisItems];
#pragma unroll
    for (int k = 0; k < kVisItems; ++k) {
      int i = base + threadIdx.x * kVisItems + k;
      const int t = i < n ? tok[i] : -1;
      flag[k] = (t >= 0 && t < kTagCount) ? 1 : 0;
      // segment starts (dag.cpp:90-98, :150-151, :155, :180): <Parallel> (Plan), <Path>,
      // <Conclusion> (Reduce), the first token, and any token right after </Parallel>.
      sflag[k] = (i < n && (t == kParOpen || t == kPathOpen || t == kConcOpen || i == 0 || tok[i - 1] == kParClose))
                     ? 1 : 0;
    }
    int stotal;
    Scan(scan_tmp).InclusiveSum(sflag, sid, stotal);
    __syncthreads();  // scan_tmp reused
    int total;
    Scan(scan_tmp).ExclusiveSum(flag, rank, total);
    const int scarry = s_seg_carry;
    if (seg_id) {
#pragma unroll
      for (int k = 0; k < kVisItems; ++k) {
        int i = base + threadIdx.x * kVisItems + k;
        if (i < n) seg_id[off + i] = scarry + sid[k] - 1;
      }
    }
    int carry = s_carry;
#pragma unroll
    for (int k = 0; k < kVisItems; ++k) {
      int i = base + threadIdx.x * kVisItems + k;
      if (i < n) {
        int r = carry + rank[k];
        if (flag[k]) {
          w.tag_idx[r] = i;
          if (r < kSmemTags) {
            s_tag_idx[r] = i;
            s_tag_kind[r] = (int8_t)tok[i];
          }
        }
        w.last_tag[i] = r + flag[k] - 1;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_carry = carry + total;
      s_seg_carry = scarry + stotal;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) s_ntags = s_carry;
  __syncthreads();
  const int T = s_ntags;

  // ---- phase 2: tag walk (single thread; O(#tags)) ----
  if (threadIdx.x == 0) {
    int err = MV_OK;
    int depth = 0;           // open frames
    int cur_pos = -1;        // position of the last token processed
    int prev_idx = -1;       // index of the previous tag
    int cur_node = -1;       // interval node applying to the current context
    int nnodes = 0;
    for (int k = 0; k < T && err == MV_OK; ++k) {
      const int idx = k < kSmemTags ? s_tag_idx[k] : w.tag_idx[k];
      const int t = k < kSmemTags ? (int)s_tag_kind[k] : tok[idx];
      const bool text_before = idx - prev_idx > 1;  // a text run sits between the tags
      int pos = cur_pos + (idx - prev_idx);
      Frame* f = depth > 0 ? &frames[depth - 1] : nullptr;
      if (!f) {
        // trajectory top level: text or <Parallel> (grammar.cpp:163-172)
        if (t != kParOpen) { err = MV_ERR_MALFORMED; break; }
      } else {
        const int ph = f->phase;
        const bool gap = ph == kAfterParOpen || ph == kAfterOutline || ph == kAfterGoal || ph == kAfterPath ||
                         ph == kAfterConclusion;
        if (gap && text_before) { err = MV_ERR_MALFORMED; break; }  // take_gap (grammar.cpp:272-282)
        switch (ph) {
          case kAfterParOpen:
            if (t != kGoalOpen) err = MV_ERR_MALFORMED;
            else f->phase = kGoalPreamble;
            break;
          case kGoalPreamble:
            if (t == kOutOpen) { f->phase = kInOutline; f->outlines++; }
            else if (f->outlines == 0) err = MV_ERR_COUNT_MISMATCH;  // grammar.cpp:195-199
            else err = MV_ERR_MALFORMED;
            break;
          case kInOutline:
            if (t != kOutClose) err = MV_ERR_MALFORMED;
            else f->phase = kAfterOutline;
            break;
          case kAfterOutline:
            if (t == kOutOpen) { f->phase = kInOutline; f->outlines++; }
            else if (t == kGoalClose) { f->phase = kAfterGoal; f->plan_end = pos; }
            else err = MV_ERR_MALFORMED;
            break;
          case kAfterGoal:
          case kAfterPath:
            if (t == kPathOpen) {
              f->paths++;
              pos = f->plan_end + 1;  // siblings share a start (dag.cpp:203-212)
              if (f->paths == 1) {
                f->first_path_idx = idx;
                cur_node = f->enclosing_node;
              } else {
                int parent = f->enclosing_node;
                int d = parent >= 0 ? (parent < kSmemTags ? s_node_w[parent] : w.nodes[parent].w) + 1 : 1;
                if (d > max_depth) { err = MV_ERR_DEPTH; break; }
                w.nodes[nnodes] = make_int4(f->first_path_idx, idx, parent, d);
                if (nnodes < kSmemTags) s_node_w[nnodes] = d;
                cur_node = nnodes++;
              }
              f->phase = kInPath;
            } else if (f->paths != f->outlines) {
              err = MV_ERR_COUNT_MISMATCH;  // grammar.cpp:228-232
            } else if (t == kConcOpen) {
              pos = f->max_path_end + 1;  // Reduce = max path end + 1
              w.single[k] = f->paths == 1;  // the Reduce segment's parents are the path tails
              cur_node = f->enclosing_node;
              f->phase = kInConclusion;
            } else {
              err = MV_ERR_MALFORMED;
            }
            break;
          case kInPath:
            if (t == kParOpen) {
              // nested block: handled below (push)
            } else if (t == kPathClose) {
              f->phase = kAfterPath;
              f->max_path_end = max(f->max_path_end, pos);
            } else {
              err = MV_ERR_MALFORMED;
            }
            break;
          case kInConclusion:
            if (t != kConcClose) err = MV_ERR_MALFORMED;
            else f->phase = kAfterConclusion;
            break;
          case kAfterConclusion:
            if (t != kParClose) err = MV_ERR_MALFORMED;
            else depth--;  // block closed (grammar.cpp:238); cur_node is the enclosing context
            break;
        }
        if (err) break;
      }
      if (t == kParOpen) {
        if (depth == kMaxFrames) { err = MV_ERR_DEPTH; break; }
        Frame nf;
        nf.phase = kAfterParOpen;
        nf.outlines = nf.paths = 0;
        nf.plan_end = nf.max_path_end = -1;
        nf.first_path_idx = -1;
        nf.enclosing_node = cur_node;
        frames[depth++] = nf;
      }
      w.tag_pos[k] = pos;
      w.tag_node[k] = cur_node;
      cur_pos = pos;
      prev_idx = idx;
    }
    if (err == MV_OK && depth > 0) {
      // end of input inside a block (grammar.cpp:250-256 `expect` at end), except the
      // count checks the parser reaches first.
      Frame* f = &frames[depth - 1];
      const bool text_after = n - 1 - prev_idx > 0;
      const bool gap = f->phase == kAfterParOpen || f->phase == kAfterOutline || f->phase == kAfterGoal ||
                       f->phase == kAfterPath || f->phase == kAfterConclusion;
      if (gap && text_after) err = MV_ERR_MALFORMED;
      else if (f->phase == kGoalPreamble && f->outlines == 0) err = MV_ERR_COUNT_MISMATCH;
      else if ((f->phase == kAfterGoal || f->phase == kAfterPath) && f->paths != f->outlines)
        err = MV_ERR_COUNT_MISMATCH;
      else err = MV_ERR_MALFORMED;
    }
    status[s] = err;
    s_err = err;
  }
  __syncthreads();
  // phase 3 (per-token positions and intervals) runs as visibility_fill_kernel over many CTAs
}

// ---- phase 3: per-token fill, one CTA per (1024-token tile, sequence) ----
// A rejected stream has no defined positions/mask (the reference throws); tags past the failure
// point were never walked, so its tiles exit.  Each token chains through its last tag's
// position / node and the node's parents: a few dependent loads, hidden across many CTAs.
constexpr int kFillThreads = 256, kFillItems = 4, kFillTile = kFillThreads * kFillItems;
__global__ void __launch_bounds__(kFillThreads) visibility_fill_kernel(const int64_t* __restrict__ offsets,
                                                                        int max_depth,
                                                                        int32_t* __restrict__ positions,
                                                                        int32_t* __restrict__ excl,
                                                                        const int32_t* __restrict__ status,
                                                                        void* ws, const int32_t* __restrict__ tokens,
                                                                        int32_t* __restrict__ targets,
                                                                        uint8_t* __restrict__ loss_mask, int tag_loss) {
  const int s = blockIdx.y;
  if (status[s] != MV_OK) return;
  const int64_t off = offsets[s];
  const int n = (int)(offsets[s + 1] - off);
  const int base = blockIdx.x * kFillTile;
  if (base >= n) return;
  SeqWs w = seq_ws(ws, off, n);
#pragma unroll
  for (int k = 0; k < kFillItems; ++k) {
    const int i = base + k * kFillThreads + threadIdx.x;
    if (i >= n) continue;
    const int lt = w.last_tag[i];
    int p, node;
    if (lt < 0) {
      p = i;
      node = -1;
    } else {
      p = w.tag_pos[lt] + (i - w.tag_idx[lt]);
      node = w.tag_node[lt];
    }
    positions[off + i] = p;
    if (targets) {
      // build_training_batch (dag.cpp:326-357): layout rows are stream order and every segment is a
      // contiguous run, so a row's target is the next token, except where the next segment is not
      // its unique chain successor: a </Path> ends its path, and only a single-path block's Reduce
      // has that path as its one parent; the last row has none.
      int tgt = -1;
      if (i + 1 < n) {
        const int nx = tokens[off + i + 1];
        tgt = nx;
        if (tokens[off + i] == kPathClose && !(nx == kConcOpen && w.single[w.last_tag[i + 1]])) tgt = -1;
      }
      targets[off + i] = tgt;
      loss_mask[off + i] = tgt >= 0 && (tag_loss || tgt >= kTagCount) ? 1 : 0;
    }
    int32_t* e = excl + (off + i) * (int64_t)max_depth * 2;
    int d = node >= 0 ? w.nodes[node].w : 0;
    for (int q = d; q < max_depth; ++q) { e[2 * q] = 0; e[2 * q + 1] = 0; }
    while (node >= 0) {
      int4 nd = w.nodes[node];
      e[2 * (nd.w - 1)] = nd.x;
      e[2 * (nd.w - 1) + 1] = nd.y;
      node = nd.z;
    }
  }
}

// Dense mask bits from intervals (dag::Mask layout, MSB-first packed).
__global__ void mask_packed_kernel(const int32_t* __restrict__ excl, int n, int D, int row0, int row1,
                                   uint8_t* __restrict__ out) {
  const int64_t nbytes = ((int64_t)(row1 - row0) * n + 7) / 8;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nbytes; b += (int64_t)gridDim.x * blockDim.x) {
    uint32_t byte = 0;
    for (int k = 0; k < 8; ++k) {
      int64_t bit = b * 8 + k;
      int i = row0 + (int)(bit / n);
      int j = (int)(bit % n);
      if (i >= row1) break;
      bool vis = j <= i;
      const int32_t* e = excl + (int64_t)i * D * 2;
      for (int q = 0; q < D && vis; ++q)
        if (j >= e[2 * q] && j < e[2 * q + 1]) vis = false;
      if (vis) byte |= 0x80u >> k;
    }
    out[b] = (uint8_t)byte;
  }
}

// Prefill tile classification: one CTA per q-tile, one thread per query row.
__global__ void tile_map_kernel(const int32_t* __restrict__ excl, int n, int D, int tile, int32_t* __restrict__ count,
                                int32_t* __restrict__ list, unsigned long long* __restrict__ visible_pairs) {
  const int qt = blockIdx.x;
  const int n_qt = (n + tile - 1) / tile;
  const int i = qt * tile + threadIdx.x;
  const bool row_ok = threadIdx.x < tile && i < n;
  int lo[8], hi[8];
  int nd = 0;
  if (row_ok) {
    for (int q = 0; q < D && q < 8; ++q) {
      int a = excl[((int64_t)i * D + q) * 2], b = excl[((int64_t)i * D + q) * 2 + 1];
      if (a < b) { lo[nd] = a; hi[nd] = b; ++nd; }
    }
  }
  unsigned long long vis_total = 0;
  int written = 0;
  for (int kt = 0; kt <= qt; ++kt) {
    int j0 = kt * tile, j1 = min(n, j0 + tile);
    bool empty = true, full = true;
    if (row_ok) {
      int last = min(j1 - 1, i);  // causal clamp
      if (j0 > i) {
        empty = true;
        full = false;
      } else {
        int vis = last - j0 + 1;
        bool touches = false;
        for (int q = 0; q < nd; ++q) {
          int a = max(lo[q], j0), b = min(hi[q], last + 1);
          if (a < b) {
            vis -= b - a;
            touches = true;
          }
        }
        for (int q = 8; q < D; ++q) {  // nesting deeper than 8: the rest from memory (intervals are disjoint)
          const int a = max(excl[((int64_t)i * D + q) * 2], j0), b = min(excl[((int64_t)i * D + q) * 2 + 1], last + 1);
          if (a < b) {
            vis -= b - a;
            touches = true;
          }
        }
        empty = vis == 0;
        full = !touches && (j1 - 1 <= i) && (j0 + tile <= n);  // tail tiles hold padding tokens
        vis_total += (unsigned long long)vis;
      }
    } else {
      full = true;  // padding rows do not force a partial tile
    }
    int all_empty = __syncthreads_and(empty ? 1 : 0);
    int all_full = __syncthreads_and(full ? 1 : 0);
    if (!all_empty && threadIdx.x == 0) {
      list[(int64_t)qt * n_qt + written] = kt | (all_full ? 0 : (1 << 30));
    }
    if (!all_empty) ++written;
  }
  if (threadIdx.x == 0) count[qt] = written;
  // block reduction of the visible-pair count
  __shared__ unsigned long long red[32];
  unsigned long long v = vis_total;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int k = 0; k < (int)(blockDim.x + 31) / 32; ++k) t += red[k];
    atomicAdd(visible_pairs, t);
  }
}


// Paired tile map for the tcgen05 prefill: one CTA per 256-row q pair (2 x 128-row tiles A and
// B), one thread per row; for every 128-token k tile it records the status of each half
// (0 skip, 1 full, 2 partial) and keeps the tile when either half needs it:
//   list[qp][k] = kt | statusA << 20 | statusB << 22.
// Paired tile map in two kernels: (A) status of every (256-row q pair, k tile) on many CTAs,
// (B) one CTA per q pair compacts the statuses into the ordered lists.
constexpr int kTm2Split = 8;        // k-tile ranges per q pair in kernel A
constexpr int kTm2Chunk = 1024;     // k tiles compacted per pass in kernel B
constexpr int kTm2Threads = 1024;

// A: thread = row of the pair (256 per CTA), CTA = (q pair, k-tile range); per warp and k tile
// the rows vote all-empty / all-full, the block combines the 4 warps of each 128-row half.
// status[qp][kt] = stA | stB << 2 (0 skip, 1 full, 2 partial).
__global__ void __launch_bounds__(256) tile_status_kernel(const int32_t* __restrict__ excl, int n, int D,
                                                          uint8_t* __restrict__ status, int stride) {
  const int qp = blockIdx.x, part = blockIdx.y;
  const int tile = 128;
  const int r = threadIdx.x, warp = r >> 5, lane = r & 31;
  const int i = qp * 256 + r;
  const bool row_ok = i < n;
  // the row's intervals in registers (fixed trip count); empty intervals never intersect
  int lo[8], hi[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    lo[q] = hi[q] = 0;
    if (row_ok && q < D) {
      lo[q] = excl[((int64_t)i * D + q) * 2];
      hi[q] = excl[((int64_t)i * D + q) * 2 + 1];
    }
  }
  const int n_kt = min((qp * 256 + 255) / tile, (n - 1) / tile) + 1;
  const int per = (n_kt + kTm2Split - 1) / kTm2Split;
  const int kt0 = part * per, kt1 = min(n_kt, kt0 + per);
  __shared__ uint8_t s_e[8][64], s_f[8][64];
  for (int base = kt0; base < kt1; base += 64) {
    const int cnt = min(64, kt1 - base);
    for (int u = 0; u < cnt; ++u) {
      const int kt = base + u;
      const int j0 = kt * tile, j1 = min(n, j0 + tile);
      bool empty = true, full = true;
      if (row_ok) {
        const int lastc = min(j1 - 1, i);
        if (j0 > i) {
          full = false;
        } else {
          int vis = lastc - j0 + 1;
          bool touches = false;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int a = max(lo[q], j0), b = min(hi[q], lastc + 1);
            if (a < b) { vis -= b - a; touches = true; }
          }
          for (int q = 8; q < D; ++q) {  // nesting deeper than 8: the rest from memory
            const int a = max(excl[((int64_t)i * D + q) * 2], j0), b = min(excl[((int64_t)i * D + q) * 2 + 1], lastc + 1);
            if (a < b) { vis -= b - a; touches = true; }
          }
          empty = vis == 0;
          full = !touches && (j1 - 1 <= i) && (j0 + tile <= n);
        }
      }
      const bool we = __all_sync(0xffffffffu, empty), wf = __all_sync(0xffffffffu, full);
      if (lane == 0) {
        s_e[warp][u] = we;
        s_f[warp][u] = wf;
      }
    }
    __syncthreads();
    if (r < cnt) {
      int st[2];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        bool all_e = true, all_f = true;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          all_e &= s_e[hh * 4 + w][r] != 0;
          all_f &= s_f[hh * 4 + w][r] != 0;
        }
        st[hh] = all_e ? 0 : (all_f ? 1 : 2);
      }
      status[(int64_t)qp * stride + base + r] = (uint8_t)(st[0] | (st[1] << 2));
    }
    __syncthreads();
  }
}

// B: ordered compactions of one q pair's statuses: the pair list, and one list per 128-row half
// holding only the k tiles whose status for that half is not 0 (with the per-half counts).
//   list[qp][k] = kt | statusA << 20 | statusB << 22.
__global__ void __launch_bounds__(kTm2Threads) tile_list_kernel(const uint8_t* __restrict__ status, int n,
                                                                int32_t* __restrict__ count,
                                                                int32_t* __restrict__ list, int stride,
                                                                int32_t* __restrict__ hcount,
                                                                int32_t* __restrict__ hlist) {
  const int qp = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int s_warp_sum[3][kTm2Threads / 32];
  const int n_kt = min((qp * 256 + 255) / 128, (n - 1) / 128) + 1;
  int written = 0, nA = 0, nB = 0;
  for (int kt0 = 0; kt0 < n_kt; kt0 += kTm2Chunk) {
    const int kt = kt0 + threadIdx.x;
    int ent = -1;
    if (kt < n_kt) {
      const int st = status[(int64_t)qp * stride + kt];
      if (st) ent = kt | ((st & 3) << 20) | ((st >> 2) << 22);
    }
    const bool kp[3] = {ent >= 0, ent >= 0 && ((ent >> 20) & 3) != 0, ent >= 0 && ((ent >> 22) & 3) != 0};
    unsigned keep[3];
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      keep[x] = __ballot_sync(0xffffffffu, kp[x]);
      if (lane == 0) s_warp_sum[x][warp] = __popc(keep[x]);
    }
    __syncthreads();
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      int base = 0, total = 0;
      for (int w = 0; w < kTm2Threads / 32; ++w) {
        const int c = s_warp_sum[x][w];
        if (w < warp) base += c;
        total += c;
      }
      const int at = base + __popc(keep[x] & ((1u << lane) - 1u));
      if (x == 0) {
        if (kp[0]) list[(int64_t)qp * stride + written + at] = ent;
        written += total;
      } else {
        if (kp[x] && hlist) hlist[(int64_t)(2 * qp + x - 1) * stride + (x == 1 ? nA : nB) + at] = ent;
        if (x == 1) nA += total;
        else nB += total;
      }
    }
    __syncthreads();  // s_warp_sum reused by the next pass
  }
  if (threadIdx.x == 0) {
    count[qp] = written;
    if (hcount) {
      hcount[2 * qp] = nA;
      hcount[2 * qp + 1] = nB;
    }
  }
}
}  // namespace
}  // namespace mv

using namespace mv;

extern "C" size_t mv_visibility_workspace_size(const int64_t* h_offsets, int32_t n_seq) {
  if (!h_offsets || n_seq <= 0) return 0;
  return (size_t)h_offsets[n_seq] * 12 * sizeof(int32_t) + 256;
}

static mv_status visibility_impl(const int32_t* d_tokens, const int64_t* h_offsets, int32_t n_seq, int32_t max_depth,
                                 int32_t* d_positions, int32_t* d_seg_id, int32_t* d_excl, int32_t* d_targets,
                                 uint8_t* d_loss_mask, int tag_loss, int32_t* d_status, void* d_workspace,
                                 size_t workspace_bytes, mv_stream_t stream) {
  if (n_seq <= 0 || !h_offsets || max_depth < 1 || !d_positions || !d_excl || !d_status)
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_visibility: bad arguments");
  if ((d_targets == nullptr) != (d_loss_mask == nullptr))
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_training_batch: targets and loss mask go together");
  if (workspace_bytes < mv_visibility_workspace_size(h_offsets, n_seq) || !d_workspace)
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_visibility: workspace too small");
  for (int s = 0; s < n_seq; ++s)
    if (h_offsets[s + 1] < h_offsets[s] || h_offsets[s + 1] - h_offsets[s] > (int64_t)INT32_MAX / 2)
      return fail(MV_ERR_INVALID_ARGUMENT, "mv_visibility: bad offsets");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int64_t* d_off = nullptr;
  MV_CUDA_TRY(cudaMallocAsync(&d_off, sizeof(int64_t) * (n_seq + 1), st));
  MV_CUDA_TRY(cudaMemcpyAsync(d_off, h_offsets, sizeof(int64_t) * (n_seq + 1), cudaMemcpyHostToDevice, st));
  visibility_kernel<<<n_seq, kVisThreads, 0, st>>>(d_tokens, d_off, max_depth, d_positions, d_seg_id, d_excl, d_status,
                                                   d_workspace);
  MV_LAUNCH_CHECK();
  int64_t max_len = 0;
  for (int s = 0; s < n_seq; ++s) max_len = std::max<int64_t>(max_len, h_offsets[s + 1] - h_offsets[s]);
  if (max_len > 0) {
    visibility_fill_kernel<<<dim3((unsigned)((max_len + kFillTile - 1) / kFillTile), n_seq), kFillThreads, 0, st>>>(
        d_off, max_depth, d_positions, d_excl, d_status, d_workspace, d_tokens, d_targets, d_loss_mask, tag_loss);
    MV_LAUNCH_CHECK();
  }
  MV_CUDA_TRY(cudaFreeAsync(d_off, st));
  return MV_OK;
}

extern "C" mv_status mv_visibility(const int32_t* d_tokens, const int64_t* h_offsets, int32_t n_seq, int32_t max_depth,
                                   int32_t* d_positions, int32_t* d_seg_id, int32_t* d_excl, int32_t* d_status,
                                   void* d_workspace, size_t workspace_bytes, mv_stream_t stream) {
  return visibility_impl(d_tokens, h_offsets, n_seq, max_depth, d_positions, d_seg_id, d_excl, nullptr, nullptr, 1,
                         d_status, d_workspace, workspace_bytes, stream);
}

extern "C" mv_status mv_training_batch(const int32_t* d_tokens, const int64_t* h_offsets, int32_t n_seq,
                                       int32_t max_depth, int32_t tag_loss, int32_t* d_positions, int32_t* d_excl,
                                       int32_t* d_targets, uint8_t* d_loss_mask, int32_t* d_status, void* d_workspace,
                                       size_t workspace_bytes, mv_stream_t stream) {
  if (!d_targets || !d_loss_mask) return fail(MV_ERR_INVALID_ARGUMENT, "mv_training_batch: null targets / loss mask");
  return visibility_impl(d_tokens, h_offsets, n_seq, max_depth, d_positions, nullptr, d_excl, d_targets, d_loss_mask,
                         tag_loss, d_status, d_workspace, workspace_bytes, stream);
}

extern "C" mv_status mv_mask_packed(const int32_t* d_excl, int32_t n, int32_t max_depth, int32_t row0, int32_t row1,
                                    uint8_t* d_out, mv_stream_t stream) {
  if (n < 0 || row0 < 0 || row1 > n || row0 > row1 || max_depth < 1)
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_mask_packed: bad arguments");
  int64_t nbytes = ((int64_t)(row1 - row0) * n + 7) / 8;
  if (nbytes == 0) return MV_OK;
  int blocks = (int)std::min<int64_t>((nbytes + 255) / 256, 148 * 16);
  mask_packed_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(d_excl, n, max_depth, row0, row1,
                                                                                  d_out);
  MV_LAUNCH_CHECK();
  return MV_OK;
}

extern "C" mv_status mv_tile_map(const int32_t* d_excl, int32_t n, int32_t max_depth, int32_t tile, int32_t* d_count,
                                 int32_t* d_list, unsigned long long* d_visible_pairs, mv_stream_t stream) {
  if (n <= 0 || tile <= 0 || tile > 1024 || (tile & 31) || max_depth < 1 || max_depth > kMaxIntervals)
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_tile_map: bad arguments");
  int n_qt = (n + tile - 1) / tile;
  tile_map_kernel<<<n_qt, tile, 0, reinterpret_cast<cudaStream_t>(stream)>>>(d_excl, n, max_depth, tile, d_count,
                                                                              d_list, d_visible_pairs);
  MV_LAUNCH_CHECK();
  return MV_OK;
}

namespace mv {
mv_status tile_map2(const int32_t* d_excl, int32_t n, int32_t max_depth, uint8_t* d_status, int32_t* d_count,
                    int32_t* d_list, int32_t stride, cudaStream_t stream, int32_t* d_hcount, int32_t* d_hlist) {
  // statuses in the caller's workspace: a byte array [n_qp][stride]
  const int n_qp = (n + 255) / 256;
  tile_status_kernel<<<dim3(n_qp, kTm2Split), 256, 0, stream>>>(d_excl, n, max_depth, d_status, stride);
  MV_LAUNCH_CHECK();
  tile_list_kernel<<<n_qp, kTm2Threads, 0, stream>>>(d_status, n, d_count, d_list, stride, d_hcount, d_hlist);
  MV_LAUNCH_CHECK();
  return MV_OK;
}
}  // namespace mv
