// kvstore.cu — K2: paged KV store with Process-stage fork and Reduce-stage merge.
//
// Reference behaviour replaced: kv::RadixStore
//   create   kvcache.cpp:90-93        extend  kvcache.cpp:149-243 (+ split_node :95-147)
//   fork     kvcache.cpp:245-252      merge   kvcache.cpp:254-289
//   release  kvcache.cpp:291-340      resolve / resolve_payloads / resolve_slots :367-397
//   stats    kvcache.cpp:353-365
//
// Parity is defined at the logical level: the same op log resolves to
// the same token and payload sequences and raises the same errors; fork and merge move
// zero payload bytes (only page-table entries). Physical slot numbering, node counts and
// radix dedup are not reproduced (a paged store does not dedup identical suffixes), so
// "physically shares the prefix" means shares by lineage (fork / extend / merge copies).
#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "store.hpp"

namespace mv {

// ---------------------------------------------------------------------------
// status plumbing
// ---------------------------------------------------------------------------
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
mv_status fail(mv_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

namespace {

constexpr uint32_t kErrNoPages = 1u;

// Pops m pages from the device free stack (CAS so a failed pop leaves the stack intact).
__device__ int pop_pages(int32_t* free_top, int m, int32_t* err) {
  int cur = *((volatile int32_t*)free_top);
  while (true) {
    if (cur < m) {
      atomicOr(err, (int)kErrNoPages);
      return -1;
    }
    int prev = atomicCAS(free_top, cur, cur - m);
    if (prev == cur) return cur - m;
    cur = prev;
  }
}

// fork / functional copy: replicate one page table into `ncopy` arena blocks.
__global__ void k_copy_table(PageRef* __restrict__ arena, int32_t* __restrict__ cum, int64_t src_off, int n,
                             const int64_t* __restrict__ dst_offs, int ncopy, int32_t* __restrict__ refcnt) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    PageRef r = arena[src_off + e];
    int32_t c = cum[src_off + e];
    for (int k = 0; k < ncopy; ++k) {
      arena[dst_offs[k] + e] = r;
      cum[dst_offs[k] + e] = c;
    }
    atomicAdd(&refcnt[r.page], ncopy);
  }
}

// merge: output entry o comes from segment j = last seg with out_begin <= o.
struct MergeSeg {
  int64_t src_off;    // arena offset of the source handle
  int32_t src_first;  // first source entry copied
  int32_t out_begin;  // first output entry of this segment
  int32_t skip;       // tokens dropped from the first copied entry (prefix overlap)
  int32_t tok_base;   // token offset of the segment in the merged sequence
  int32_t prefix_len; // tokens of the merge prefix in source coordinates (0 for the prefix itself)
  int32_t pad;
};

__global__ void k_merge(PageRef* __restrict__ arena, int32_t* __restrict__ cum, const MergeSeg* __restrict__ segs,
                        int nseg, int n_out, int64_t dst_off, int32_t* __restrict__ refcnt) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < n_out; o += gridDim.x * blockDim.x) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (segs[mid].out_begin <= o) lo = mid;
      else hi = mid - 1;
    }
    const MergeSeg sg = segs[lo];
    int64_t se = sg.src_off + sg.src_first + (o - sg.out_begin);
    PageRef r = arena[se];
    if (o == sg.out_begin && sg.skip > 0) r = make_ref(r.page, ref_begin(r) + sg.skip, ref_count(r) - sg.skip);
    arena[dst_off + o] = r;
    cum[dst_off + o] = sg.tok_base + max(cum[se] - sg.prefix_len, 0);
    atomicAdd(&refcnt[r.page], 1);
  }
}

__device__ __forceinline__ uint32_t slot_of(const PageRef* arena, const int32_t* cum, int64_t off, int n_entries,
                                            int t) {
  int lo = 0, hi = n_entries - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (cum[off + mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  PageRef r = arena[off + lo];
  return (uint32_t)r.page * kPageTokens + (uint32_t)(ref_begin(r) + (t - cum[off + lo]));
}

// merge precondition (kvcache.cpp:268-274): every branch shares the prefix slot for slot.
struct BranchDesc {
  int64_t off;
  int32_t n_entries;
  int32_t pad;
};
__global__ void k_merge_check(const PageRef* __restrict__ arena, const int32_t* __restrict__ cum, int64_t p_off,
                              int p_entries, int p_len, const BranchDesc* __restrict__ br, int nb,
                              int32_t* __restrict__ bad) {
  int64_t total = (int64_t)p_len * nb;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    int b = (int)(x / p_len);
    int t = (int)(x % p_len);
    uint32_t sp = slot_of(arena, cum, p_off, p_entries, t);
    uint32_t sb = slot_of(arena, cum, br[b].off, br[b].n_entries, t);
    if (sp != sb) atomicOr(bad, 1);
  }
}

// release: one page reference per table entry; pages reaching zero go back on the stack.
struct TableDesc {
  int64_t off;
  int32_t n;
  int32_t pad;
};
__global__ void k_release(const PageRef* __restrict__ arena, const TableDesc* __restrict__ tabs, int32_t* refcnt,
                          int32_t* free_stack, int32_t* free_top) {
  const TableDesc td = tabs[blockIdx.y];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < td.n; e += gridDim.x * blockDim.x) {
    int p = arena[td.off + e].page;
    if (atomicSub(&refcnt[p], 1) == 1) {
      int idx = atomicAdd(free_top, 1);
      free_stack[idx] = p;
    }
  }
}

// Bulk append to one handle: step 1 (single thread) pops pages and edits the table.
struct AppendPlan {
  int64_t tail_idx;   // arena index of the current tail entry (in-place fill), -1 if none
  int64_t new_idx;    // arena index of the first new entry
  int32_t fill;       // tokens written in place into the tail page
  int32_t new_pages;  // pages to pop
  int32_t n;          // tokens appended
  int32_t tok_base;   // tokens before the append
};
__global__ void k_append_table(PageRef* __restrict__ arena, int32_t* __restrict__ cum, AppendPlan pl,
                               int32_t* __restrict__ refcnt, int32_t* __restrict__ free_stack,
                               int32_t* __restrict__ free_top, int32_t* __restrict__ err,
                               int32_t* __restrict__ page_out /*[new_pages]*/, int32_t* __restrict__ tail_out /*2*/) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (pl.fill > 0) {
    PageRef r = arena[pl.tail_idx];
    tail_out[0] = r.page;
    tail_out[1] = ref_begin(r) + ref_count(r);
    arena[pl.tail_idx] = make_ref(r.page, ref_begin(r), ref_count(r) + pl.fill);
  }
  if (pl.new_pages > 0) {
    int base = pop_pages(free_top, pl.new_pages, err);
    int left = pl.n - pl.fill;
    for (int k = 0; k < pl.new_pages; ++k) {
      int p = base >= 0 ? free_stack[base + k] : 0;
      int cnt = min(kPageTokens, left - k * kPageTokens);
      page_out[k] = base >= 0 ? p : -1;
      if (base >= 0) {
        arena[pl.new_idx + k] = make_ref(p, 0, cnt);
        cum[pl.new_idx + k] = pl.tok_base + pl.fill + k * kPageTokens;
        refcnt[p] = 1;
      }
    }
  }
}

// step 2: per token, write slot token ids, payload records and (optionally) K/V.
__device__ __forceinline__ void rope8(uint4& v, int pos, int chunk, const double* inv) {
  // 8 dims = 4 interleaved pairs, pair index t = chunk*4 + j (toy_model.cpp:30-41)
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float c, s;
    rope_cs(pos, inv[chunk * 4 + j], c, s);
    float2 ab = __bfloat1622float2(h[j]);
    h[j] = __floats2bfloat162_rn(ab.x * c - ab.y * s, ab.x * s + ab.y * c);
  }
}

__device__ __forceinline__ void write_kv_token(__nv_bfloat16* kp, __nv_bfloat16* vp, int64_t page, int slot,
                                               int kv_heads, int64_t npages, const __nv_bfloat16* k,
                                               const __nv_bfloat16* v, int pos, const double* inv, int lane,
                                               int nlanes, int hd, int first = 0) {
  // kv_heads * hd / 8 chunks of 8 dims (from chunk `first`); K rotated, V verbatim; stored chunk-swizzled.
  const int lg = hd == 128 ? 4 : 3;  // log2 chunks per head
  for (int j = first + lane; j < (kv_heads << lg); j += nlanes) {
    int h = j >> lg, c = j & ((1 << lg) - 1);
    size_t dst = kv_page_head_offset(page, h, npages, hd) + (size_t)kv_chunk_offset(slot, c, hd);
    uint4 kk = *reinterpret_cast<const uint4*>(k + (size_t)h * hd + c * 8);
    rope8(kk, pos, c, inv);
    *reinterpret_cast<uint4*>(kp + dst) = kk;
    *reinterpret_cast<uint4*>(vp + dst) = *reinterpret_cast<const uint4*>(v + (size_t)h * hd + c * 8);
  }
}

__global__ void k_append_data(AppendPlan pl, const int32_t* __restrict__ page_out, const int32_t* __restrict__ tail,
                              const int32_t* __restrict__ tokens, int32_t* __restrict__ slot_tok,
                              const uint8_t* __restrict__ rec_in, uint8_t* __restrict__ records, int rec_bytes,
                              const int32_t* __restrict__ pos, const __nv_bfloat16* __restrict__ k,
                              const __nv_bfloat16* __restrict__ v, __nv_bfloat16* kp, __nv_bfloat16* vp, int kv_heads,
                              int64_t npages, const RopeTable rt) {
  __shared__ double s_inv[kMaxHeadDim / 2];
  const double* inv = rope_stage(rt, s_inv);
  // one warp per token
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (warp >= pl.n) return;
  int t = warp;
  int64_t page;
  int slot;
  if (t < pl.fill) {
    page = tail[0];
    slot = tail[1] + t;
  } else {
    int q = t - pl.fill;
    page = page_out[q / kPageTokens];
    slot = q % kPageTokens;
  }
  if (page < 0) return;  // out of pages; the sticky error is reported by the host
  int64_t gslot = page * kPageTokens + slot;
  if (lane == 0 && tokens) slot_tok[gslot] = tokens[t];
  if (rec_in && rec_bytes > 0)
    for (int b = lane; b < rec_bytes; b += 32) records[gslot * rec_bytes + b] = rec_in[(int64_t)t * rec_bytes + b];
  if (k && v)
    write_kv_token(kp, vp, page, slot, kv_heads, npages, k + (size_t)t * kv_heads * rt.hd,
                   v + (size_t)t * kv_heads * rt.hd, pos ? pos[t] : 0, inv, lane, 32, rt.hd);
}

// Engine fast path: one token per handle, in place (one warp per handle, 4 per CTA).
// Descriptors of up to kDescInline tokens travel in the launch's parameter space (no separate
// host->device copy in the stream); larger batches use an uploaded array.
constexpr int kDescInline = 240;
struct TokDescInline {
  TokDesc d[kDescInline];
};

// One warp per token.  The token's K/V chunks (<= 4 per lane for <= 8 kv heads) are loaded and
// rotated before lane 0's page-table update resolves the destination, so the two latency
// chains overlap; the stores follow the shuffle of (page, slot).
__device__ __forceinline__ void append_one_warp(const TokDesc td, int i, PageRef* __restrict__ arena,
                                                int32_t* __restrict__ cum, const int32_t* __restrict__ tokens,
                                                int32_t* __restrict__ slot_tok, int32_t* __restrict__ refcnt,
                                                int32_t* __restrict__ free_stack, int32_t* __restrict__ free_top,
                                                int32_t* __restrict__ err, const int32_t* __restrict__ pos,
                                                const __nv_bfloat16* __restrict__ k,
                                                const __nv_bfloat16* __restrict__ v, __nv_bfloat16* kp,
                                                __nv_bfloat16* vp, int kv_heads, int64_t npages,
                                                const double* inv, int hd) {
  const int lane = threadIdx.x & 31;
  // programmatic launch: the inputs (k, v, positions, tokens) may be produced by the kernel
  // this one overlaps (e.g. the caller's projection GEMM), so nothing is read before this wait;
  // only the launch latency and the frequency staging overlap the predecessor
  pdl_wait();
  const bool kv = k && v;
  const int lg = hd == 128 ? 4 : 3;  // log2 16-byte chunks per head
  const int nch = kv ? kv_heads << lg : 0;  // 16-byte chunks of the token's K (and V)
  const __nv_bfloat16* kt = kv ? k + (size_t)i * kv_heads * hd : nullptr;
  const __nv_bfloat16* vt = kv ? v + (size_t)i * kv_heads * hd : nullptr;
  uint4 kk[4], vv[4];
  const int p = kv ? __ldg(pos + i) : 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j = lane + 32 * u;
    if (j < nch) {
      kk[u] = __ldg(reinterpret_cast<const uint4*>(kt) + j);
      vv[u] = __ldg(reinterpret_cast<const uint4*>(vt) + j);
    }
  }
  int page = -1, slot = 0;
  if (lane == 0) {
    if (td.fresh) {
      // the host reserved this page (PagedStore::reserve_pages), so the pop cannot fail; a failure
      // is a reservation bug, reported through err at the next reservation sync
      int old = atomicSub(free_top, 1);
      if (old >= 1) {
        page = free_stack[old - 1];
        arena[td.idx] = make_ref(page, 0, 1);
        cum[td.idx] = td.cumv;
        refcnt[page] = 1;
      } else {
        atomicAdd(free_top, 1);
        atomicOr(err, (int)kErrNoPages);
      }
    } else {
      PageRef r = arena[td.idx];
      page = r.page;
      slot = ref_begin(r) + ref_count(r);
      arena[td.idx] = make_ref(r.page, ref_begin(r), ref_count(r) + 1);
    }
    if (page >= 0 && tokens) slot_tok[(int64_t)page * kPageTokens + slot] = tokens[i];
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
    if (lane + 32 * u < nch) rope8(kk[u], p, (lane + 32 * u) & ((1 << lg) - 1), inv);
  page = __shfl_sync(0xffffffffu, page, 0);
  slot = __shfl_sync(0xffffffffu, slot, 0);
  if (page < 0 || !kv) return;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j = lane + 32 * u;
    if (j < nch) {
      const size_t dst = kv_page_head_offset(page, j >> lg, npages, hd) + (size_t)kv_chunk_offset(slot, j & ((1 << lg) - 1), hd);
      *reinterpret_cast<uint4*>(kp + dst) = kk[u];
      *reinterpret_cast<uint4*>(vp + dst) = vv[u];
    }
  }
  if (nch > 128)  // more than 128 chunks (8 kv heads at hd 128): the rest after the destination is known
    write_kv_token(kp, vp, page, slot, kv_heads, npages, kt, vt, p, inv, lane, 32, hd, 128);
}

__global__ void k_append_one(PageRef* __restrict__ arena, int32_t* __restrict__ cum, const TokDesc* __restrict__ d,
                             int n, const int32_t* __restrict__ tokens, int32_t* __restrict__ slot_tok,
                             int32_t* __restrict__ refcnt, int32_t* __restrict__ free_stack,
                             int32_t* __restrict__ free_top, int32_t* __restrict__ err, const int32_t* __restrict__ pos,
                             const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v,
                             __nv_bfloat16* kp, __nv_bfloat16* vp, int kv_heads, int64_t npages, const RopeTable rt) {
  __shared__ double s_inv[kMaxHeadDim / 2];
  const double* inv = rope_stage(rt, s_inv);
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  append_one_warp((threadIdx.x & 31) == 0 ? d[i] : TokDesc{0, 0, 0}, i, arena, cum, tokens, slot_tok, refcnt,
                  free_stack, free_top, err, pos, k, v, kp, vp, kv_heads, npages, inv, rt.hd);
}
__global__ void k_append_one_inline(PageRef* __restrict__ arena, int32_t* __restrict__ cum, const TokDescInline d,
                                    int n, const int32_t* __restrict__ tokens, int32_t* __restrict__ slot_tok,
                                    int32_t* __restrict__ refcnt, int32_t* __restrict__ free_stack,
                                    int32_t* __restrict__ free_top, int32_t* __restrict__ err,
                                    const int32_t* __restrict__ pos, const __nv_bfloat16* __restrict__ k,
                                    const __nv_bfloat16* __restrict__ v, __nv_bfloat16* kp, __nv_bfloat16* vp,
                                    int kv_heads, int64_t npages, const RopeTable rt) {
  // the RoPE pre-pass after this kernel may launch now: it waits (griddepcontrol.wait) for this
  // grid to complete before touching anything, and only then releases decode_tc
  pdl_launch_dependents();
  __shared__ double s_inv[kMaxHeadDim / 2];
  const double* inv = rope_stage(rt, s_inv);
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  append_one_warp(d.d[i], i, arena, cum, tokens, slot_tok, refcnt, free_stack, free_top, err, pos, k, v, kp, vp,
                  kv_heads, npages, inv, rt.hd);
}

// K/V of the last token of each handle (for layers > the one written at append).
__global__ void k_write_last(const PageRef* __restrict__ arena, const int64_t* __restrict__ idx,
                             const int32_t* __restrict__ pos, const __nv_bfloat16* __restrict__ k,
                             const __nv_bfloat16* __restrict__ v, __nv_bfloat16* kp, __nv_bfloat16* vp, int kv_heads,
                             int64_t npages, const RopeTable rt) {
  __shared__ double s_inv[kMaxHeadDim / 2];
  const double* inv = rope_stage(rt, s_inv);
  const int i = blockIdx.x;
  PageRef r = arena[idx[i]];
  int slot = ref_begin(r) + ref_count(r) - 1;
  write_kv_token(kp, vp, r.page, slot, kv_heads, npages, k + (size_t)i * kv_heads * rt.hd,
                 v + (size_t)i * kv_heads * rt.hd, pos[i], inv, threadIdx.x, blockDim.x, rt.hd);
}

// K/V of tokens [first, first + n) of one handle for one layer (multi-layer bulk prefill: layer 0 goes
// with append_many, the other layers through this), one warp per token; the token's slot comes from
// the handle's entries by binary search over the prefix sums.
__global__ void k_write_range(const PageRef* __restrict__ arena, const int32_t* __restrict__ cum, int64_t off,
                              int n_entries, int first, int n, const int32_t* __restrict__ pos,
                              const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v,
                              __nv_bfloat16* kp, __nv_bfloat16* vp, int kv_heads, int64_t npages, const RopeTable rt) {
  __shared__ double s_inv[kMaxHeadDim / 2];
  const double* inv = rope_stage(rt, s_inv);
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= n) return;
  const int t = first + w;
  int lo = 0, hi = n_entries - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (cum[off + mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  const PageRef r = arena[off + lo];
  write_kv_token(kp, vp, r.page, ref_begin(r) + (t - cum[off + lo]), kv_heads, npages,
                 k + (size_t)w * kv_heads * rt.hd, v + (size_t)w * kv_heads * rt.hd, pos ? pos[w] : 0, inv,
                 lane, 32, rt.hd);
}

// resolve / resolve_payloads / resolve_slots / gather_kv: one thread block per entry.
__global__ void k_resolve(const PageRef* __restrict__ arena, const int32_t* __restrict__ cum, int64_t off, int n,
                          const int32_t* __restrict__ slot_tok, const uint8_t* __restrict__ records, int rec_bytes,
                          int32_t* __restrict__ tok_out, uint8_t* __restrict__ rec_out, uint32_t* __restrict__ slot_out,
                          const __nv_bfloat16* __restrict__ kp, const __nv_bfloat16* __restrict__ vp, int kv_heads,
                          int64_t npages, __nv_bfloat16* __restrict__ k_out, __nv_bfloat16* __restrict__ v_out,
                          int hd) {
  for (int e = blockIdx.x; e < n; e += gridDim.x) {
    PageRef r = arena[off + e];
    int c0 = cum[off + e];
    int b = ref_begin(r), cnt = ref_count(r);
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
      int64_t gslot = (int64_t)r.page * kPageTokens + b + t;
      if (tok_out) tok_out[c0 + t] = slot_tok[gslot];
      if (slot_out) slot_out[c0 + t] = (uint32_t)gslot;
    }
    if (rec_out)
      for (int x = threadIdx.x; x < cnt * rec_bytes; x += blockDim.x)
        rec_out[(int64_t)c0 * rec_bytes + x] = records[((int64_t)r.page * kPageTokens + b) * rec_bytes + x];
    if (k_out)
      for (int x = threadIdx.x; x < cnt * kv_heads * (hd / 8); x += blockDim.x) {
        const int ch = hd / 8;
        int t = x / (kv_heads * ch), h = (x / ch) % kv_heads, c = x % ch;
        int slot = b + t;
        size_t src = kv_page_head_offset(r.page, h, npages, hd) + (size_t)kv_chunk_offset(slot, c, hd);
        size_t dst = ((size_t)(c0 + t) * kv_heads + h) * hd + c * 8;
        *reinterpret_cast<uint4*>(k_out + dst) = *reinterpret_cast<const uint4*>(kp + src);
        *reinterpret_cast<uint4*>(v_out + dst) = *reinterpret_cast<const uint4*>(vp + src);
      }
  }
}

// stats: mark referenced slots, then count.
__global__ void k_mark(const PageRef* __restrict__ arena, const TableDesc* __restrict__ tabs,
                       uint32_t* __restrict__ bitmap) {
  const TableDesc td = tabs[blockIdx.y];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < td.n; e += gridDim.x * blockDim.x) {
    PageRef r = arena[td.off + e];
    uint32_t bits = ((1u << ref_count(r)) - 1u) << ref_begin(r);  // 16 slots -> 16 bits of a word half
    atomicOr(&bitmap[r.page >> 1], bits << ((r.page & 1) * 16));
  }
}
__global__ void k_count(const uint32_t* __restrict__ bitmap, int64_t words, const int32_t* __restrict__ refcnt,
                        int pages, unsigned long long* __restrict__ out /*[3]: slots, pages_in_use, refsum*/) {
  unsigned long long a = 0, b = 0, c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x)
    a += __popc(bitmap[i]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < pages; i += (int64_t)gridDim.x * blockDim.x) {
    b += refcnt[i] > 0;
    c += (unsigned long long)refcnt[i];
  }
  atomicAdd(&out[0], a);
  atomicAdd(&out[1], b);
  atomicAdd(&out[2], c);
}

// Ascending stack: a bulk pop of m pages (k_append_table takes stack[top - m .. top)) hands out an
// ascending run of page ids, so a fresh pool stores a bulk append contiguously (16 KiB decode copies).
__global__ void k_init_free(int32_t* free_stack, int n, int32_t* free_top) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) free_stack[i] = i;
  if (blockIdx.x == 0 && threadIdx.x == 0) *free_top = n;
}

int grid_for(int64_t n, int threads) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 8)); }

int32_t pow2_cap(int32_t need) {
  int32_t c = 16;
  while (c < need) c <<= 1;
  return c;
}

}  // namespace

// ---------------------------------------------------------------------------
// PagedStore
// ---------------------------------------------------------------------------
PagedStore::PagedStore(const mv_kv_config& cfg) : cfg_(cfg) {
  if (cfg_.table_entries <= 0) cfg_.table_entries = 4 * (int64_t)cfg_.num_pages + 65536;
  if (cfg_.rope_base <= 0) cfg_.rope_base = 10000.0;
  rope_ = make_rope_table(cfg_.rope_base, cfg_.head_dim > 0 ? cfg_.head_dim : kHeadDim);
}

PagedStore::~PagedStore() {
  cudaStreamSynchronize(stream_);
  cudaFree(d_arena);
  cudaFree(d_cum);
  cudaFree(d_refcnt_);
  cudaFree(d_free_);
  cudaFree(d_free_top_);
  cudaFree(d_err_);
  cudaFree(d_slot_tok_);
  cudaFree(d_records_);
  for (auto* p : k_planes_) cudaFree(p);
  for (auto* p : v_planes_) cudaFree(p);
  for (auto* p : dscratch_) cudaFree(p);
  for (auto& sg : stage_)
    for (int k = 0; k < 2; ++k) {
      if (sg.buf[k]) cudaFreeHost(sg.buf[k]);
      if (sg.ev[k]) cudaEventDestroy(sg.ev[k]);
    }
  if (pinned_) cudaFreeHost(pinned_);
  destroy_plan(plan);
}

mv_status PagedStore::init() {
  if (cfg_.num_pages <= 0 || cfg_.record_bytes < 0 || cfg_.layers < 0 || cfg_.kv_heads < 0)
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_kv_store_create: bad config");
  if (cfg_.kv_heads > 0 && (!head_dim_supported(cfg_.head_dim) || cfg_.layers < 1))
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_kv_store_create: attention plane needs head_dim 64 or 128 and layers >= 1");
  const int64_t slots = (int64_t)cfg_.num_pages * kPageTokens;
  MV_CUDA_TRY(cudaMalloc(&d_arena, sizeof(PageRef) * cfg_.table_entries));
  MV_CUDA_TRY(cudaMalloc(&d_cum, sizeof(int32_t) * cfg_.table_entries));
  MV_CUDA_TRY(cudaMalloc(&d_refcnt_, sizeof(int32_t) * cfg_.num_pages));
  MV_CUDA_TRY(cudaMemset(d_refcnt_, 0, sizeof(int32_t) * cfg_.num_pages));
  MV_CUDA_TRY(cudaMalloc(&d_free_, sizeof(int32_t) * cfg_.num_pages));
  MV_CUDA_TRY(cudaMalloc(&d_free_top_, sizeof(int32_t)));
  MV_CUDA_TRY(cudaMalloc(&d_err_, sizeof(int32_t)));
  MV_CUDA_TRY(cudaMemset(d_err_, 0, sizeof(int32_t)));
  MV_CUDA_TRY(cudaMalloc(&d_slot_tok_, sizeof(int32_t) * slots));
  if (cfg_.record_bytes > 0) MV_CUDA_TRY(cudaMalloc(&d_records_, (size_t)slots * cfg_.record_bytes));
  if (cfg_.kv_heads > 0) {
    size_t plane = (size_t)slots * cfg_.kv_heads * cfg_.head_dim * sizeof(__nv_bfloat16);
    for (int l = 0; l < cfg_.layers; ++l) {
      __nv_bfloat16 *k = nullptr, *v = nullptr;
      MV_CUDA_TRY(cudaMalloc(&k, plane));
      MV_CUDA_TRY(cudaMalloc(&v, plane));
      // zero once: masked slots of a ragged page must never hold NaN bit patterns (0 * NaN)
      MV_CUDA_TRY(cudaMemsetAsync(k, 0, plane, stream_));
      MV_CUDA_TRY(cudaMemsetAsync(v, 0, plane, stream_));
      k_planes_.push_back(k);
      v_planes_.push_back(v);
    }
  }
  k_init_free<<<grid_for(cfg_.num_pages, 256), 256, 0, stream_>>>(d_free_, cfg_.num_pages, d_free_top_);
  MV_LAUNCH_CHECK();
  MV_CUDA_TRY(cudaStreamSynchronize(stream_));
  free_lb_ = cfg_.num_pages;
  return MV_OK;
}

HandleRec* PagedStore::find(uint64_t h) {
  auto it = handles_.find(h);
  return it == handles_.end() ? nullptr : &it->second;
}

static mv_status unknown(uint64_t h) {
  // kvcache.cpp:16-20: unknown handles are reported as DoubleRelease.
  return fail(MV_ERR_DOUBLE_RELEASE, "handle " + std::to_string(h) + " is unknown or already released");
}

int64_t PagedStore::arena_alloc(int32_t need, int32_t* cap_out) {
  int32_t cap = pow2_cap(std::max(need, 1));
  auto it = free_blocks_.find(cap);
  if (it != free_blocks_.end() && !it->second.empty()) {
    int64_t off = it->second.back();
    it->second.pop_back();
    *cap_out = cap;
    return off;
  }
  if (arena_top_ + cap > cfg_.table_entries) return -1;
  int64_t off = arena_top_;
  arena_top_ += cap;
  *cap_out = cap;
  return off;
}

void PagedStore::arena_free(int64_t off, int32_t cap) {
  if (cap > 0) free_blocks_[cap].push_back(off);
}

mv_status PagedStore::ensure_cap(HandleRec& r, int32_t need) {
  if (need <= r.cap) return MV_OK;
  int32_t cap;
  int64_t off = arena_alloc(need * 2, &cap);
  if (off < 0) return fail(MV_ERR_CAPACITY, "page-table arena exhausted");
  if (r.n_entries() > 0) {
    MV_CUDA_TRY(cudaMemcpyAsync(d_arena + off, d_arena + r.arena_off, sizeof(PageRef) * r.n_entries(),
                                cudaMemcpyDeviceToDevice, stream_));
    MV_CUDA_TRY(cudaMemcpyAsync(d_cum + off, d_cum + r.arena_off, sizeof(int32_t) * r.n_entries(),
                                cudaMemcpyDeviceToDevice, stream_));
  }
  arena_free(r.arena_off, r.cap);
  r.arena_off = off;
  r.cap = cap;
  return MV_OK;
}

uint64_t PagedStore::register_handle(HandleRec rec) {
  uint64_t id = next_handle_++;
  logical_ += rec.n_tokens();
  rec.version = 1;
  handles_.emplace(id, std::move(rec));
  return id;
}

void* PagedStore::device_scratch(size_t bytes, int slot) {
  if ((int)dscratch_.size() <= slot) {
    dscratch_.resize(slot + 1, nullptr);
    dscratch_bytes_.resize(slot + 1, 0);
  }
  if (dscratch_bytes_[slot] < bytes) {
    if (dscratch_[slot]) cudaFreeAsync(dscratch_[slot], stream_);
    size_t nb = std::max<size_t>(bytes, 4096);
    nb = std::max(nb, dscratch_bytes_[slot] * 2);
    if (cudaMallocAsync(&dscratch_[slot], nb, stream_) != cudaSuccess) {
      dscratch_[slot] = nullptr;
      dscratch_bytes_[slot] = 0;
      return nullptr;
    }
    dscratch_bytes_[slot] = nb;
  }
  return dscratch_[slot];
}

// Host -> device staging of small per-call arrays (page-table descriptors): copied into one of two
// pinned buffers per slot (ping-pong, guarded by an event), so the async copy neither drains the
// stream (as a pageable source would) nor races a copy still in flight.
mv_status PagedStore::upload(const void* host, size_t bytes, void** dev_out, int slot) {
  void* d = device_scratch(bytes, slot);
  if (!d) return fail(MV_ERR_CUDA, "device scratch allocation failed");
  if (bytes) {
    if ((int)stage_.size() <= slot) stage_.resize(slot + 1);
    Stage& sg = stage_[slot];
    const int k = sg.next;
    sg.next ^= 1;
    if (sg.ev[k]) MV_CUDA_TRY(cudaEventSynchronize(sg.ev[k]));
    else MV_CUDA_TRY(cudaEventCreateWithFlags(&sg.ev[k], cudaEventDisableTiming));
    if (sg.bytes[k] < bytes) {
      if (sg.buf[k]) cudaFreeHost(sg.buf[k]);
      sg.bytes[k] = std::max<size_t>(bytes, 4096);
      MV_CUDA_TRY(cudaMallocHost(&sg.buf[k], sg.bytes[k]));
    }
    std::memcpy(sg.buf[k], host, bytes);
    MV_CUDA_TRY(cudaMemcpyAsync(d, sg.buf[k], bytes, cudaMemcpyHostToDevice, stream_));
    MV_CUDA_TRY(cudaEventRecord(sg.ev[k], stream_));
  }
  *dev_out = d;
  return MV_OK;
}

void* PagedStore::pinned(size_t bytes) {
  if (pinned_bytes_ < bytes) {
    if (pinned_) {
      cudaStreamSynchronize(stream_);
      cudaFreeHost(pinned_);
    }
    pinned_bytes_ = std::max<size_t>(bytes, 1 << 16);
    if (cudaMallocHost(&pinned_, pinned_bytes_) != cudaSuccess) {
      pinned_ = nullptr;
      pinned_bytes_ = 0;
    }
  }
  return pinned_;
}

mv_status PagedStore::reserve_pages(int64_t m, const char* what) {
  if (m <= 0) return MV_OK;
  if (m > free_lb_) {
    // the bound says the pool may run out: wait for the queued pops / releases and re-read the stack
    int32_t top = 0, e = 0;
    MV_CUDA_TRY(cudaMemcpyAsync(&top, d_free_top_, sizeof top, cudaMemcpyDeviceToHost, stream_));
    MV_CUDA_TRY(cudaMemcpyAsync(&e, d_err_, sizeof e, cudaMemcpyDeviceToHost, stream_));
    MV_CUDA_TRY(cudaStreamSynchronize(stream_));
    if (e) {
      MV_CUDA_TRY(cudaMemsetAsync(d_err_, 0, sizeof(int32_t), stream_));
      return fail(MV_ERR_CUDA, std::string(what) + ": internal error: a device page pop failed");
    }
    free_lb_ = top;
    if (m > free_lb_)
      return fail(MV_ERR_CAPACITY, std::string(what) + ": store capacity of " +
                                       std::to_string((int64_t)cfg_.num_pages * kPageTokens) + " tokens exceeded");
  }
  free_lb_ -= m;
  return MV_OK;
}

mv_status PagedStore::create(uint64_t* out) {
  HandleRec r;
  int32_t cap;
  int64_t off = arena_alloc(16, &cap);
  if (off < 0) return fail(MV_ERR_CAPACITY, "page-table arena exhausted");
  r.arena_off = off;
  r.cap = cap;
  *out = register_handle(std::move(r));
  return MV_OK;
}

mv_status PagedStore::fork(uint64_t h, int32_t n, uint64_t* out) {
  if (n < 0) return fail(MV_ERR_INVALID_ARGUMENT, "fork: n < 0");
  HandleRec* src = find(h);
  if (!src) return unknown(h);
  if (n == 0) return MV_OK;
  const uint64_t group = next_group_++;
  std::vector<int64_t> offs(n);
  std::vector<HandleRec> kids(n);
  for (int k = 0; k < n; ++k) {
    HandleRec& c = kids[k];
    int32_t cap;
    int64_t off = arena_alloc(src->n_entries() + 1, &cap);
    if (off < 0) {
      for (int j = 0; j < k; ++j) arena_free(kids[j].arena_off, kids[j].cap);
      return fail(MV_ERR_CAPACITY, "page-table arena exhausted");
    }
    c.arena_off = off;
    c.cap = cap;
    c.cum = src->cum;
    c.tail_room = 0;  // the parent keeps the in-place budget of the shared tail page
    c.lineage = src->lineage;
    c.lineage.push_back({group, src->n_entries(), src->n_tokens(), h, src->version});
    offs[k] = off;
  }
  if (src->n_entries() > 0) {
    void* d_offs;
    if (mv_status st = upload(offs.data(), sizeof(int64_t) * n, &d_offs, 0)) return st;
    k_copy_table<<<grid_for(src->n_entries(), 256), 256, 0, stream_>>>(
        d_arena, d_cum, src->arena_off, src->n_entries(), (const int64_t*)d_offs, n, d_refcnt_);
    MV_LAUNCH_CHECK();
  }
  for (int k = 0; k < n; ++k) out[k] = register_handle(std::move(kids[k]));
  return MV_OK;
}

mv_status PagedStore::extend(uint64_t h, const int32_t* tokens, int64_t n, const void* payloads, uint64_t* out) {
  if (n < 0) return fail(MV_ERR_INVALID_ARGUMENT, "extend: negative token count");
  HandleRec* src = find(h);
  if (!src) return unknown(h);
  HandleRec r;
  const int32_t fill = (int32_t)std::min<int64_t>(src->tail_room, n);
  const int64_t rest = n - fill;
  const int32_t new_pages = (int32_t)((rest + kPageTokens - 1) / kPageTokens);
  // capacity first (kvcache.cpp:37-41 throws before the store changes)
  if (mv_status st = reserve_pages(new_pages, "extend")) return st;
  int32_t cap;
  int64_t off = arena_alloc(src->n_entries() + new_pages + 1, &cap);
  if (off < 0) {
    unreserve_pages(new_pages);
    return fail(MV_ERR_CAPACITY, "page-table arena exhausted");
  }
  r.cum = src->cum;
  r.lineage = src->lineage;
  r.arena_off = off;
  r.cap = cap;
  // 1) copy the source table (shares every page; one ref per copied entry)
  if (src->n_entries() > 0) {
    void* d_offs;
    if (mv_status st = upload(&off, sizeof(int64_t), &d_offs, 0)) return st;
    k_copy_table<<<grid_for(src->n_entries(), 256), 256, 0, stream_>>>(d_arena, d_cum, src->arena_off,
                                                                     src->n_entries(), (const int64_t*)d_offs, 1,
                                                                     d_refcnt_);
    MV_LAUNCH_CHECK();
  }
  // 2) in-place fill of the tail page (the new handle takes over the tail budget), then new pages
  AppendPlan pl;
  pl.tail_idx = fill > 0 ? off + src->n_entries() - 1 : -1;
  pl.new_idx = off + src->n_entries();
  pl.fill = fill;
  pl.new_pages = new_pages;
  pl.n = (int32_t)n;
  pl.tok_base = (int32_t)src->n_tokens();
  if (n > 0) {
    void *d_tok = nullptr, *d_rec = nullptr;
    // (a CUDA failure from here on leaves the store unusable, as any CUDA error does)
    if (mv_status st = upload(tokens, sizeof(int32_t) * n, &d_tok, 1)) return st;
    if (payloads && cfg_.record_bytes > 0)
      if (mv_status st = upload(payloads, (size_t)n * cfg_.record_bytes, &d_rec, 2)) return st;
    int32_t* d_pages = (int32_t*)device_scratch(sizeof(int32_t) * (new_pages + 2), 3);
    if (!d_pages) return fail(MV_ERR_CUDA, "scratch allocation failed");
    k_append_table<<<1, 32, 0, stream_>>>(d_arena, d_cum, pl, d_refcnt_, d_free_, d_free_top_, d_err_, d_pages,
                                          d_pages + new_pages);
    MV_LAUNCH_CHECK();
    int64_t threads = n * 32;
    k_append_data<<<(int)((threads + 255) / 256), 256, 0, stream_>>>(
        pl, d_pages, d_pages + new_pages, (const int32_t*)d_tok, d_slot_tok_, (const uint8_t*)d_rec, d_records_,
        cfg_.record_bytes, nullptr, nullptr, nullptr, nullptr, nullptr, cfg_.kv_heads, cfg_.num_pages, rope_);
    MV_LAUNCH_CHECK();
    for (int64_t t = 0; t < fill; ++t) r.cum.back()++;
    for (int32_t k = 0; k < new_pages; ++k) {
      int64_t cnt = std::min<int64_t>(kPageTokens, rest - (int64_t)k * kPageTokens);
      r.cum.push_back(r.cum.back() + (int32_t)cnt);
    }
    if (new_pages > 0) {
      r.tail_room = kPageTokens - (int32_t)(rest - (int64_t)(new_pages - 1) * kPageTokens);
    } else {
      r.tail_room = src->tail_room - fill;
    }
    src->tail_room = 0;
  } else {
    // zero-token extend: a second handle on the same tail; nobody may fill it in place now
    r.tail_room = 0;
    src->tail_room = 0;
  }
  *out = register_handle(std::move(r));
  return MV_OK;
}

mv_status PagedStore::merge(uint64_t prefix, const uint64_t* branches, int32_t nb, uint64_t* out) {
  HandleRec* p = find(prefix);
  if (!p) return unknown(prefix);
  if (nb < 0) return fail(MV_ERR_INVALID_ARGUMENT, "merge: negative branch count");
  const int64_t plen = p->n_tokens();
  std::vector<MergeSeg> segs;
  std::vector<BranchDesc> bdesc;
  HandleRec r;
  r.cum = p->cum;
  r.lineage = p->lineage;
  segs.push_back({p->arena_off, 0, 0, 0, 0, 0, 0});
  int32_t out_n = p->n_entries();
  bool all_proven = true;
  for (int b = 0; b < nb; ++b) {
    HandleRec* br = find(branches[b]);
    if (!br) return unknown(branches[b]);
    if (br->n_tokens() < plen)
      return fail(MV_ERR_NOT_DESCENDANT, "branch shorter than the merge prefix");  // kvcache.cpp:262-265
    // host proof of the slot-identity precondition: the branch descends from a fork of `prefix`
    // taken while `prefix` was exactly as it is now (its version is unchanged since)
    bool proven = br == p;
    for (auto& lg : br->lineage)
      if (lg.src == prefix && lg.src_version == p->version && lg.tokens == plen) proven = true;
    all_proven = all_proven && proven;
    bdesc.push_back({br->arena_off, br->n_entries(), 0});
    if (br->n_tokens() == plen) continue;
    // first branch entry holding token `plen`
    int32_t k = (int32_t)(std::upper_bound(br->cum.begin(), br->cum.end(), (int32_t)plen) - br->cum.begin()) - 1;
    int32_t skip = (int32_t)(plen - br->cum[k]);
    MergeSeg sg;
    sg.src_off = br->arena_off;
    sg.src_first = k;
    sg.out_begin = out_n;
    sg.skip = skip;
    sg.tok_base = (int32_t)r.n_tokens();
    sg.prefix_len = (int32_t)plen;
    sg.pad = 0;
    segs.push_back(sg);
    for (int32_t e = k; e < br->n_entries(); ++e) {
      int32_t cnt = br->cum[e + 1] - std::max<int32_t>(br->cum[e], (int32_t)plen);
      r.cum.push_back(r.cum.back() + cnt);
    }
    out_n += br->n_entries() - k;
  }
  // slot-identity precondition (kvcache.cpp:268-274) for branches the lineage does not prove:
  // checked on the device, synchronously (merge throws like the reference)
  if (nb > 0 && plen > 0 && !all_proven) {
    void* d_b;
    if (mv_status st = upload(bdesc.data(), sizeof(BranchDesc) * bdesc.size(), &d_b, 4)) return st;
    int32_t* d_bad = (int32_t*)device_scratch(sizeof(int32_t), 5);
    MV_CUDA_TRY(cudaMemsetAsync(d_bad, 0, sizeof(int32_t), stream_));
    k_merge_check<<<grid_for(plen * nb, 256), 256, 0, stream_>>>(d_arena, d_cum, p->arena_off, p->n_entries(),
                                                                (int)plen, (const BranchDesc*)d_b, nb, d_bad);
    MV_LAUNCH_CHECK();
    int32_t bad = 0;
    MV_CUDA_TRY(cudaMemcpyAsync(&bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost, stream_));
    MV_CUDA_TRY(cudaStreamSynchronize(stream_));
    if (bad) return fail(MV_ERR_NOT_DESCENDANT, "branch does not share the merge prefix");
  }
  int32_t cap;
  int64_t off = arena_alloc(out_n + 1, &cap);
  if (off < 0) return fail(MV_ERR_CAPACITY, "page-table arena exhausted");
  r.arena_off = off;
  r.cap = cap;
  r.tail_room = 0;  // the merged tail page stays with the last branch (sealed for the merge)
  if (out_n > 0) {
    void* d_s;
    if (mv_status st = upload(segs.data(), sizeof(MergeSeg) * segs.size(), &d_s, 6)) return st;
    k_merge<<<grid_for(out_n, 256), 256, 0, stream_>>>(d_arena, d_cum, (const MergeSeg*)d_s, (int)segs.size(), out_n,
                                                        off, d_refcnt_);
    MV_LAUNCH_CHECK();
  }
  *out = register_handle(std::move(r));
  return MV_OK;
}

mv_status PagedStore::release(uint64_t h) {
  auto it = handles_.find(h);
  if (it == handles_.end()) return unknown(h);
  HandleRec& r = it->second;
  if (r.n_entries() > 0) {
    TableDesc td{r.arena_off, r.n_entries(), 0};
    void* d_t;
    if (mv_status st = upload(&td, sizeof td, &d_t, 7)) return st;
    dim3 grid(grid_for(r.n_entries(), 256), 1);
    k_release<<<grid, 256, 0, stream_>>>(d_arena, (const TableDesc*)d_t, d_refcnt_, d_free_, d_free_top_);
    MV_LAUNCH_CHECK();
  }
  logical_ -= r.n_tokens();
  arena_free(r.arena_off, r.cap);
  handles_.erase(it);
  return MV_OK;
}

mv_status PagedStore::length(uint64_t h, int64_t* out) {
  HandleRec* r = find(h);
  if (!r) return unknown(h);
  *out = r->n_tokens();
  return MV_OK;
}

mv_status PagedStore::stats(mv_kv_stats* out) {
  std::vector<TableDesc> tabs;
  for (auto& [id, r] : handles_)
    if (r.n_entries() > 0) tabs.push_back({r.arena_off, r.n_entries(), 0});
  const int64_t words = ((int64_t)cfg_.num_pages + 1) / 2;
  uint32_t* bitmap = (uint32_t*)device_scratch(sizeof(uint32_t) * words + 64, 8);
  if (!bitmap) return fail(MV_ERR_CUDA, "scratch allocation failed");
  unsigned long long* cnt = (unsigned long long*)(bitmap + words + (words & 1));
  MV_CUDA_TRY(cudaMemsetAsync(bitmap, 0, sizeof(uint32_t) * words + 64, stream_));
  if (!tabs.empty()) {
    void* d_t;
    if (mv_status st = upload(tabs.data(), sizeof(TableDesc) * tabs.size(), &d_t, 7)) return st;
    int maxn = 0;
    for (auto& t : tabs) maxn = std::max(maxn, t.n);
    dim3 grid(grid_for(maxn, 256), (unsigned)tabs.size());
    k_mark<<<grid, 256, 0, stream_>>>(d_arena, (const TableDesc*)d_t, bitmap);
    MV_LAUNCH_CHECK();
  }
  k_count<<<grid_for(std::max<int64_t>(words, cfg_.num_pages), 256), 256, 0, stream_>>>(bitmap, words, d_refcnt_,
                                                                                       cfg_.num_pages, cnt);
  MV_LAUNCH_CHECK();
  unsigned long long host[3] = {0, 0, 0};
  int32_t top = 0;
  MV_CUDA_TRY(cudaMemcpyAsync(host, cnt, sizeof host, cudaMemcpyDeviceToHost, stream_));
  MV_CUDA_TRY(cudaMemcpyAsync(&top, d_free_top_, sizeof top, cudaMemcpyDeviceToHost, stream_));
  MV_CUDA_TRY(cudaStreamSynchronize(stream_));
  free_lb_ = top;  // exact after the sync
  out->physical_tokens_stored = host[0];
  out->logical_tokens_reachable = (uint64_t)logical_;
  out->bytes_copied_on_last_op = 0;
  out->live_handles = handles_.size();
  out->node_count = host[1];
  out->total_refcount = host[2];
  out->free_pages = (uint64_t)top;
  return MV_OK;
}

mv_status PagedStore::resolve(uint64_t h, int32_t* tokens, void* payloads, uint32_t* slots) {
  HandleRec* r = find(h);
  if (!r) return unknown(h);
  const int64_t len = r->n_tokens();
  if (len == 0) return MV_OK;
  size_t tb = tokens ? sizeof(int32_t) * len : 0;
  size_t pb = (payloads && cfg_.record_bytes > 0) ? (size_t)len * cfg_.record_bytes : 0;
  size_t sb = slots ? sizeof(uint32_t) * len : 0;
  uint8_t* d = (uint8_t*)device_scratch(tb + pb + sb + 64, 9);
  if (!d) return fail(MV_ERR_CUDA, "scratch allocation failed");
  int32_t* d_tok = tb ? (int32_t*)d : nullptr;
  uint32_t* d_slot = sb ? (uint32_t*)(d + tb) : nullptr;
  uint8_t* d_rec = pb ? d + tb + sb : nullptr;
  k_resolve<<<std::min(r->n_entries(), 148 * 16), 128, 0, stream_>>>(
      d_arena, d_cum, r->arena_off, r->n_entries(), d_slot_tok_, d_records_, cfg_.record_bytes, d_tok, d_rec, d_slot,
      nullptr, nullptr, cfg_.kv_heads, (int64_t)cfg_.num_pages, nullptr, nullptr, rope_.hd);
  MV_LAUNCH_CHECK();
  if (tb) MV_CUDA_TRY(cudaMemcpyAsync(tokens, d_tok, tb, cudaMemcpyDeviceToHost, stream_));
  if (sb) MV_CUDA_TRY(cudaMemcpyAsync(slots, d_slot, sb, cudaMemcpyDeviceToHost, stream_));
  if (pb) MV_CUDA_TRY(cudaMemcpyAsync(payloads, d_rec, pb, cudaMemcpyDeviceToHost, stream_));
  MV_CUDA_TRY(cudaStreamSynchronize(stream_));
  return MV_OK;
}

mv_status PagedStore::append(const uint64_t* hs, int32_t n, const int32_t* d_tokens, const int32_t* d_pos,
                             int32_t layer, const void* d_k, const void* d_v) {
  if (n <= 0) return n == 0 ? MV_OK : fail(MV_ERR_INVALID_ARGUMENT, "append: n < 0");
  if ((d_k || d_v) && (cfg_.kv_heads == 0 || layer < 0 || layer >= cfg_.layers || !d_pos))
    return fail(MV_ERR_INVALID_ARGUMENT, "append: no attention plane for this layer / positions missing");
  // pass 1 validates everything before any state changes: unknown handles, a handle listed twice
  // (two warps would extend the same entry), table capacity, and the pages this call pops
  std::vector<HandleRec*>& recs = append_recs_;
  recs.resize(n);
  const uint64_t stamp = ++call_stamp_;
  int64_t fresh = 0;
  for (int i = 0; i < n; ++i) {
    HandleRec* r = find(hs[i]);
    if (!r) return unknown(hs[i]);
    if (r->stamp == stamp) return fail(MV_ERR_INVALID_ARGUMENT, "append: handle " + std::to_string(hs[i]) + " listed twice");
    r->stamp = stamp;
    recs[i] = r;
    if (r->tail_room == 0) {
      ++fresh;
      if (mv_status st = ensure_cap(*r, r->n_entries() + 1)) return st;  // moves the table only
    }
  }
  if (mv_status st = reserve_pages(fresh, "append")) return st;
  // pass 2 commits the host metadata (cannot fail)
  std::vector<TokDesc>& desc = append_desc_;
  desc.resize(n);
  for (int i = 0; i < n; ++i) {
    HandleRec* r = recs[i];
    if (r->tail_room > 0) {
      desc[i] = {r->arena_off + r->n_entries() - 1, 0, 0};
      r->tail_room--;
      r->cum.back()++;
    } else {
      desc[i] = {r->arena_off + r->n_entries(), 1, (int32_t)r->n_tokens()};
      r->cum.push_back(r->cum.back() + 1);
      r->tail_room = kPageTokens - 1;
    }
    r->version++;
  }
  logical_ += n;
  __nv_bfloat16* kpl = d_k ? k_planes_[layer] : nullptr;
  __nv_bfloat16* vpl = d_k ? v_planes_[layer] : nullptr;
  if (n <= kDescInline) {  // descriptors ride in the launch parameters: no copy in the stream
    TokDescInline inl;
    std::memcpy(inl.d, desc.data(), sizeof(TokDesc) * n);
    // programmatic dependent launch: launch latency and frequency staging overlap the
    // previous kernel (every input read follows griddepcontrol.wait)
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((n + 3) / 4);
    lc.blockDim = dim3(128);
    lc.stream = stream_;
    lc.attrs = pdl;
    lc.numAttrs = 1;
    MV_CUDA_TRY(cudaLaunchKernelEx(&lc, k_append_one_inline, d_arena, d_cum, inl, n, d_tokens, d_slot_tok_, d_refcnt_,
                                   d_free_, d_free_top_, d_err_, d_pos, (const __nv_bfloat16*)d_k,
                                   (const __nv_bfloat16*)d_v, kpl, vpl, (int)cfg_.kv_heads, (int64_t)cfg_.num_pages,
                                   rope_));
  } else {
    void* d_desc;
    if (mv_status st = upload(desc.data(), sizeof(TokDesc) * n, &d_desc, 10)) return st;
    k_append_one<<<(n + 3) / 4, 128, 0, stream_>>>(d_arena, d_cum, (const TokDesc*)d_desc, n, d_tokens, d_slot_tok_,
                                                   d_refcnt_, d_free_, d_free_top_, d_err_, d_pos,
                                                   (const __nv_bfloat16*)d_k, (const __nv_bfloat16*)d_v, kpl, vpl,
                                                   cfg_.kv_heads, (int64_t)cfg_.num_pages, rope_);
  }
  MV_LAUNCH_CHECK();
  return MV_OK;
}

mv_status PagedStore::write_last(const uint64_t* hs, int32_t n, const int32_t* d_pos, int32_t layer, const void* d_k,
                                 const void* d_v) {
  if (n <= 0) return n == 0 ? MV_OK : fail(MV_ERR_INVALID_ARGUMENT, "write_last: n < 0");
  if (cfg_.kv_heads == 0 || layer < 0 || layer >= cfg_.layers || !d_k || !d_v || !d_pos)
    return fail(MV_ERR_INVALID_ARGUMENT, "write_last: bad layer or buffers");
  std::vector<int64_t> idx(n);
  for (int i = 0; i < n; ++i) {
    HandleRec* r = find(hs[i]);
    if (!r) return unknown(hs[i]);
    if (r->n_entries() == 0) return fail(MV_ERR_INVALID_ARGUMENT, "write_last: empty handle");
    idx[i] = r->arena_off + r->n_entries() - 1;
  }
  void* d_idx;
  if (mv_status st = upload(idx.data(), sizeof(int64_t) * n, &d_idx, 11)) return st;
  k_write_last<<<n, 128, 0, stream_>>>(d_arena, (const int64_t*)d_idx, d_pos, (const __nv_bfloat16*)d_k,
                                       (const __nv_bfloat16*)d_v, k_planes_[layer], v_planes_[layer], cfg_.kv_heads,
                                       (int64_t)cfg_.num_pages, rope_);
  MV_LAUNCH_CHECK();
  return MV_OK;
}

mv_status PagedStore::append_many(uint64_t h, int64_t n, const int32_t* d_tokens, const int32_t* d_pos, int32_t layer,
                                  const void* d_k, const void* d_v) {
  HandleRec* r = find(h);
  if (!r) return unknown(h);
  if (n <= 0) return n == 0 ? MV_OK : fail(MV_ERR_INVALID_ARGUMENT, "append_many: n < 0");
  if ((d_k || d_v) && (cfg_.kv_heads == 0 || layer < 0 || layer >= cfg_.layers || !d_pos))
    return fail(MV_ERR_INVALID_ARGUMENT, "append_many: no attention plane for this layer / positions missing");
  const int32_t fill = (int32_t)std::min<int64_t>(r->tail_room, n);
  const int64_t rest = n - fill;
  const int32_t new_pages = (int32_t)((rest + kPageTokens - 1) / kPageTokens);
  if (mv_status st = reserve_pages(new_pages, "append_many")) return st;
  if (mv_status st = ensure_cap(*r, r->n_entries() + new_pages + 1)) {
    unreserve_pages(new_pages);
    return st;
  }
  AppendPlan pl;
  pl.tail_idx = fill > 0 ? r->arena_off + r->n_entries() - 1 : -1;
  pl.new_idx = r->arena_off + r->n_entries();
  pl.fill = fill;
  pl.new_pages = new_pages;
  pl.n = (int32_t)n;
  pl.tok_base = (int32_t)r->n_tokens();
  int32_t* d_pages = (int32_t*)device_scratch(sizeof(int32_t) * (new_pages + 2), 3);
  if (!d_pages) return fail(MV_ERR_CUDA, "scratch allocation failed");
  k_append_table<<<1, 32, 0, stream_>>>(d_arena, d_cum, pl, d_refcnt_, d_free_, d_free_top_, d_err_, d_pages,
                                        d_pages + new_pages);
  MV_LAUNCH_CHECK();
  int64_t threads = n * 32;
  k_append_data<<<(int)((threads + 255) / 256), 256, 0, stream_>>>(
      pl, d_pages, d_pages + new_pages, d_tokens, d_slot_tok_, nullptr, d_records_, cfg_.record_bytes, d_pos,
      (const __nv_bfloat16*)d_k, (const __nv_bfloat16*)d_v, d_k ? k_planes_[layer] : nullptr,
      d_k ? v_planes_[layer] : nullptr, cfg_.kv_heads, (int64_t)cfg_.num_pages, rope_);
  MV_LAUNCH_CHECK();
  r->cum.back() += fill;
  for (int32_t k = 0; k < new_pages; ++k) {
    int64_t cnt = std::min<int64_t>(kPageTokens, rest - (int64_t)k * kPageTokens);
    r->cum.push_back(r->cum.back() + (int32_t)cnt);
  }
  r->tail_room = new_pages > 0 ? kPageTokens - (int32_t)(rest - (int64_t)(new_pages - 1) * kPageTokens)
                               : r->tail_room - fill;
  r->version++;
  logical_ += n;
  return MV_OK;
}

mv_status PagedStore::write_range(uint64_t h, int64_t first, int64_t n, const int32_t* d_pos, int32_t layer,
                                  const void* d_k, const void* d_v) {
  HandleRec* r = find(h);
  if (!r) return unknown(h);
  if (cfg_.kv_heads == 0 || layer < 0 || layer >= cfg_.layers || !d_k || !d_v)
    return fail(MV_ERR_INVALID_ARGUMENT, "write_range: no attention plane for this layer / null K, V");
  if (first < 0 || n < 0 || first + n > r->n_tokens())
    return fail(MV_ERR_INVALID_ARGUMENT, "write_range: token range outside the handle");
  if (n == 0) return MV_OK;
  const int64_t threads = n * 32;
  k_write_range<<<(int)((threads + 255) / 256), 256, 0, stream_>>>(
      d_arena, d_cum, r->arena_off, r->n_entries(), (int)first, (int)n, d_pos, (const __nv_bfloat16*)d_k,
      (const __nv_bfloat16*)d_v, k_planes_[layer], v_planes_[layer], cfg_.kv_heads, (int64_t)cfg_.num_pages, rope_);
  MV_LAUNCH_CHECK();
  return MV_OK;
}

mv_status PagedStore::gather_kv(uint64_t h, int32_t layer, void* d_k, void* d_v) {
  HandleRec* r = find(h);
  if (!r) return unknown(h);
  if (cfg_.kv_heads == 0 || layer < 0 || layer >= cfg_.layers)
    return fail(MV_ERR_INVALID_ARGUMENT, "gather_kv: no attention plane for this layer");
  if (r->n_entries() == 0) return MV_OK;
  k_resolve<<<std::min(r->n_entries(), 148 * 16), 128, 0, stream_>>>(
      d_arena, d_cum, r->arena_off, r->n_entries(), d_slot_tok_, d_records_, cfg_.record_bytes, nullptr, nullptr,
      nullptr, k_planes_[layer], v_planes_[layer], cfg_.kv_heads, (int64_t)cfg_.num_pages, (__nv_bfloat16*)d_k,
      (__nv_bfloat16*)d_v, rope_.hd);
  MV_LAUNCH_CHECK();
  return MV_OK;
}

}  // namespace mv

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
using mv::fail;

#define STORE_OR_FAIL(s)                                                            \
  do {                                                                              \
    if (!(s) || !(s)->impl) return fail(MV_ERR_INVALID_ARGUMENT, "null store");     \
  } while (0)

extern "C" const char* mv_last_error(void) { return mv::g_last_error.c_str(); }
extern "C" const char* mv_version(void) { return "multiverse-b200 0.1 (sm_100a)"; }

extern "C" mv_status mv_kv_store_create(const mv_kv_config* cfg, mv_kv_store** out) {
  if (!cfg || !out) return fail(MV_ERR_INVALID_ARGUMENT, "null argument");
  auto* impl = new mv::PagedStore(*cfg);
  mv_status st = impl->init();
  if (st != MV_OK) {
    delete impl;
    return st;
  }
  *out = new mv_kv_store{impl};
  return MV_OK;
}

extern "C" mv_status mv_kv_store_destroy(mv_kv_store* s) {
  if (!s) return MV_OK;
  delete s->impl;
  delete s;
  return MV_OK;
}

extern "C" mv_status mv_kv_set_stream(mv_kv_store* s, mv_stream_t stream) {
  STORE_OR_FAIL(s);
  s->impl->set_stream(reinterpret_cast<cudaStream_t>(stream));
  return MV_OK;
}

extern "C" mv_status mv_kv_planes(mv_kv_store* s, int32_t layer, void** d_k, void** d_v) {
  STORE_OR_FAIL(s);
  if (layer < 0 || layer >= s->impl->cfg().layers || s->impl->cfg().kv_heads == 0)
    return fail(MV_ERR_INVALID_ARGUMENT, "no attention plane for this layer");
  *d_k = s->impl->k_planes()[layer];
  *d_v = s->impl->v_planes()[layer];
  return MV_OK;
}

extern "C" mv_status mv_kv_create(mv_kv_store* s, uint64_t* out) {
  STORE_OR_FAIL(s);
  return s->impl->create(out);
}
extern "C" mv_status mv_kv_extend(mv_kv_store* s, uint64_t h, const int32_t* tokens, int64_t n, const void* payloads,
                                  uint64_t* out) {
  STORE_OR_FAIL(s);
  return s->impl->extend(h, tokens, n, payloads, out);
}
extern "C" mv_status mv_kv_fork(mv_kv_store* s, uint64_t h, int32_t n, uint64_t* out) {
  STORE_OR_FAIL(s);
  return s->impl->fork(h, n, out);
}
extern "C" mv_status mv_kv_merge(mv_kv_store* s, uint64_t prefix, const uint64_t* branches, int32_t nb, uint64_t* out) {
  STORE_OR_FAIL(s);
  return s->impl->merge(prefix, branches, nb, out);
}
extern "C" mv_status mv_kv_release(mv_kv_store* s, uint64_t h) {
  STORE_OR_FAIL(s);
  return s->impl->release(h);
}
extern "C" mv_status mv_kv_length(mv_kv_store* s, uint64_t h, int64_t* out) {
  STORE_OR_FAIL(s);
  return s->impl->length(h, out);
}
extern "C" mv_status mv_kv_stats_get(mv_kv_store* s, mv_kv_stats* out) {
  STORE_OR_FAIL(s);
  return s->impl->stats(out);
}
extern "C" mv_status mv_kv_resolve(mv_kv_store* s, uint64_t h, int32_t* tokens) {
  STORE_OR_FAIL(s);
  return s->impl->resolve(h, tokens, nullptr, nullptr);
}
extern "C" mv_status mv_kv_resolve_payloads(mv_kv_store* s, uint64_t h, void* out) {
  STORE_OR_FAIL(s);
  return s->impl->resolve(h, nullptr, out, nullptr);
}
extern "C" mv_status mv_kv_resolve_slots(mv_kv_store* s, uint64_t h, uint32_t* slots) {
  STORE_OR_FAIL(s);
  return s->impl->resolve(h, nullptr, nullptr, slots);
}
extern "C" mv_status mv_kv_append(mv_kv_store* s, const uint64_t* hs, int32_t n, const int32_t* d_tokens,
                                  const int32_t* d_pos, int32_t layer, const void* d_k, const void* d_v) {
  STORE_OR_FAIL(s);
  return s->impl->append(hs, n, d_tokens, d_pos, layer, d_k, d_v);
}
extern "C" mv_status mv_kv_write_last(mv_kv_store* s, const uint64_t* hs, int32_t n, const int32_t* d_pos,
                                      int32_t layer, const void* d_k, const void* d_v) {
  STORE_OR_FAIL(s);
  return s->impl->write_last(hs, n, d_pos, layer, d_k, d_v);
}
extern "C" mv_status mv_kv_append_many(mv_kv_store* s, uint64_t h, int64_t n, const int32_t* d_tokens,
                                       const int32_t* d_pos, int32_t layer, const void* d_k, const void* d_v) {
  STORE_OR_FAIL(s);
  return s->impl->append_many(h, n, d_tokens, d_pos, layer, d_k, d_v);
}
extern "C" mv_status mv_kv_write_range(mv_kv_store* s, uint64_t h, int64_t first, int64_t n, const int32_t* d_positions,
                                       int32_t layer, const void* d_k, const void* d_v) {
  STORE_OR_FAIL(s);
  return s->impl->write_range(h, first, n, d_positions, layer, d_k, d_v);
}
extern "C" mv_status mv_kv_gather_kv(mv_kv_store* s, uint64_t h, int32_t layer, void* d_k, void* d_v) {
  STORE_OR_FAIL(s);
  return s->impl->gather_kv(h, layer, d_k, d_v);
}
