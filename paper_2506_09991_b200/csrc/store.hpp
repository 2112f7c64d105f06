// store.hpp — host control plane of the paged KV store (K2).
//
// Split of responsibilities:
//   device (source of truth for identity): page pool, per-page refcounts, free-page stack,
//     page-table arena (PageRef entries + per-entry token prefix sums), token id per slot,
//     payload records, bf16 K/V planes.  Fork / merge / extend / append / release are
//     kernels that edit those arrays; page ids never travel to the host.
//   host (shapes only): per handle the arena block, entry count, token prefix sums,
//     the in-place-append budget of its tail page, and its fork lineage (for cascade
//     decode planning).  Every host decision is deterministic and needs no device sync.
#pragma once

#include <cstdint>
#include <map>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace mv {

struct HandleRec {
  int64_t arena_off = 0;             // first entry in the device arena
  int32_t cap = 0;                   // arena block capacity (entries)
  std::vector<int32_t> cum{0};       // cum[k] = tokens before entry k; size n_entries + 1
  int32_t tail_room = 0;             // slots of the tail page this handle may fill in place
  // Fork lineage: (share-group id, entry boundary, token boundary). Entries [0, boundary)
  // are identical in every handle holding the group (SURVEY.md §7 H3 cascade).
  // src / src_version: the forked handle and its version at the fork; while that handle is
  // unchanged, its whole sequence is a slot-identical prefix of every holder (merge precondition
  // proven on the host, kvcache.cpp:268-274).
  struct Lineage {
    uint64_t group;
    int32_t entries;
    int64_t tokens;
    uint64_t src;
    uint64_t src_version;
  };
  std::vector<Lineage> lineage;
  uint64_t version = 0;              // bumps whenever the table changes (decode plan cache)
  uint64_t stamp = 0;                // per-call mark (duplicate handles in one append)

  int32_t n_entries() const { return (int32_t)cum.size() - 1; }
  int64_t n_tokens() const { return cum.back(); }
};

// Engine fast-path append descriptor (one token per handle, kvstore.cu).
struct TokDesc {
  int64_t idx;     // arena index of the entry to extend / create
  int32_t fresh;   // 1 -> pop a page and create entry (page,0,1); 0 -> grow entry in place
  int32_t cumv;    // cum value for a fresh entry
};

struct DecodePlanCache;  // decode.cu
void destroy_plan(DecodePlanCache* p);

class PagedStore {
 public:
  explicit PagedStore(const mv_kv_config& cfg);
  ~PagedStore();
  mv_status init();

  const mv_kv_config& cfg() const { return cfg_; }
  const RopeTable& rope() const { return rope_; }
  cudaStream_t stream() const { return stream_; }
  void set_stream(cudaStream_t s) { stream_ = s; }

  mv_status create(uint64_t* out);
  mv_status extend(uint64_t h, const int32_t* tokens, int64_t n, const void* payloads, uint64_t* out);
  mv_status fork(uint64_t h, int32_t n, uint64_t* out);
  mv_status merge(uint64_t prefix, const uint64_t* branches, int32_t nb, uint64_t* out);
  mv_status release(uint64_t h);
  mv_status length(uint64_t h, int64_t* out);
  mv_status stats(mv_kv_stats* out);
  mv_status resolve(uint64_t h, int32_t* tokens, void* payloads, uint32_t* slots);

  mv_status append(const uint64_t* hs, int32_t n, const int32_t* d_tokens, const int32_t* d_pos, int32_t layer,
                   const void* d_k, const void* d_v);
  mv_status write_last(const uint64_t* hs, int32_t n, const int32_t* d_pos, int32_t layer, const void* d_k,
                       const void* d_v);
  mv_status append_many(uint64_t h, int64_t n, const int32_t* d_tokens, const int32_t* d_pos, int32_t layer,
                        const void* d_k, const void* d_v);
  mv_status write_range(uint64_t h, int64_t first, int64_t n, const int32_t* d_pos, int32_t layer, const void* d_k,
                        const void* d_v);
  mv_status gather_kv(uint64_t h, int32_t layer, void* d_k, void* d_v);

  HandleRec* find(uint64_t h);
  // device arrays (read by the attention kernels)
  PageRef* d_arena = nullptr;
  int32_t* d_cum = nullptr;
  __nv_bfloat16** k_planes() { return k_planes_.data(); }
  __nv_bfloat16** v_planes() { return v_planes_.data(); }

  // scratch helpers shared with decode.cu
  void* pinned(size_t bytes);                 // host staging (grows; ordered by stream sync points)
  void* device_scratch(size_t bytes, int slot);
  // Page reservation (CacheError::CapacityExceeded, kvcache.cpp:37-41): every page-popping call
  // reserves its pages against a host lower bound of the device free stack BEFORE it touches any
  // host or device state. Releases only raise the device count, so the bound stays valid without a
  // sync; only when it says the pool may run out does the store synchronise and re-read the stack.
  mv_status reserve_pages(int64_t m, const char* what);
  void unreserve_pages(int64_t m) { free_lb_ += m; }
  DecodePlanCache* plan = nullptr;

 private:
  int64_t arena_alloc(int32_t need, int32_t* cap_out);
  void arena_free(int64_t off, int32_t cap);
  mv_status ensure_cap(HandleRec& r, int32_t need);
  uint64_t register_handle(HandleRec rec);
  mv_status upload(const void* host, size_t bytes, void** dev_out, int slot);

  mv_kv_config cfg_;
  RopeTable rope_;
  cudaStream_t stream_ = nullptr;
  int32_t* d_refcnt_ = nullptr;
  int32_t* d_free_ = nullptr;      // free-page stack
  int32_t* d_free_top_ = nullptr;  // stack size (device scalar)
  int32_t* d_err_ = nullptr;       // device error bits (1 = a page pop failed: a reservation bug)
  int64_t free_lb_ = 0;            // host lower bound of the device free-page count
  uint64_t call_stamp_ = 0;
  std::vector<HandleRec*> append_recs_;  // per-call scratch of append (kept to avoid reallocation)
  std::vector<TokDesc> append_desc_;
  int32_t* d_slot_tok_ = nullptr;  // token id per slot
  uint8_t* d_records_ = nullptr;   // record_bytes per slot
  std::vector<__nv_bfloat16*> k_planes_, v_planes_;
  std::unordered_map<uint64_t, HandleRec> handles_;
  uint64_t next_handle_ = 1;
  uint64_t next_group_ = 1;
  std::map<int32_t, std::vector<int64_t>> free_blocks_;  // arena blocks by capacity
  int64_t arena_top_ = 0;
  int64_t logical_ = 0;
  // staging
  void* pinned_ = nullptr;
  size_t pinned_bytes_ = 0;
  std::vector<void*> dscratch_;
  struct Stage {
    void* buf[2] = {nullptr, nullptr};
    size_t bytes[2] = {0, 0};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int next = 0;
  };
  std::vector<Stage> stage_;  // pinned ping-pong staging per upload slot
  std::vector<size_t> dscratch_bytes_;
};

}  // namespace mv

struct mv_kv_store {
  mv::PagedStore* impl;
};
