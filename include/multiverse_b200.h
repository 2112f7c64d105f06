/*
 * multiverse_b200.h — C-ABI of the B200-native Multiverse Attention hot path.
 *
 * This is the drop-in boundary for the reference's proj/core hot-path interface
 * (SURVEY.md §8b). Every entry point cites the reference interface it replaces.
 * Plain pointers, sizes and status codes only: no torch or C++ types.
 *
 * Conventions
 *   - Every function returns mv_status; on failure mv_last_error() (thread-local) holds
 *     a message. Status codes mirror the reference's exception kinds:
 *       CacheError::Kind      kvcache.hpp:32-41  -> MV_ERR_UNKNOWN_HANDLE .. MV_ERR_NOT_DESCENDANT
 *       ParseError::Kind      grammar.hpp:136-152 -> MV_ERR_MALFORMED, MV_ERR_COUNT_MISMATCH
 *       std::invalid_argument (toy_model.cpp:47-51, kvcache.cpp:153-156) -> MV_ERR_INVALID_ARGUMENT
 *     The reference reports an unknown handle as DoubleRelease (kvcache.cpp:16-20); so do we.
 *   - "d_" pointers are caller-owned device memory; "h_" pointers are host memory.
 *   - mv_stream_t is ABI-identical to cudaStream_t (NULL = legacy default stream).
 *   - Tag-stream encoding: tok::Tokenizer ids (tokenizer.cpp:56-63): ids 0..9 are the ten
 *     control tags in TagKind order (grammar.hpp:34-46), ids >= 10 are text.
 */
#ifndef MULTIVERSE_B200_H_
#define MULTIVERSE_B200_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MV_API __attribute__((visibility("default")))
#else
#define MV_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* mv_stream_t;

typedef enum {
  MV_OK = 0,
  MV_ERR_UNKNOWN_HANDLE = 1,   /* CacheError::UnknownHandle */
  MV_ERR_DOUBLE_RELEASE = 2,   /* CacheError::DoubleRelease (also unknown handles, kvcache.cpp:16-20) */
  MV_ERR_CAPACITY = 3,         /* CacheError::CapacityExceeded */
  MV_ERR_NOT_DESCENDANT = 4,   /* CacheError::BranchNotDescendant */
  MV_ERR_MALFORMED = 5,        /* ParseError::MalformedStructure */
  MV_ERR_COUNT_MISMATCH = 6,   /* ParseError::CountMismatch */
  MV_ERR_INVALID_ARGUMENT = 7, /* std::invalid_argument */
  MV_ERR_CUDA = 8,             /* CUDA runtime failure */
  MV_ERR_DEPTH = 9             /* nesting deeper than the caller's exclusion capacity */
} mv_status;

/* Thread-local message for the last non-OK status. */
MV_API const char* mv_last_error(void);
/* Library version string and the compiled device architecture ("sm_100a"). */
MV_API const char* mv_version(void);

/* ======================================================================== */
/* K1 — structured mask and position-id builder                              */
/* ======================================================================== */
/*
 * Replaces dag::build_dag + dag::assign_positions + dag::build_mask
 * (dag.hpp:94-110, dag.cpp:117-263) and the parse errors of grammar::parse
 * (grammar.cpp:156-294), for a batch of tag streams in one launch.
 *
 *   d_tokens   int32 ids, all sequences concatenated; sequence s is
 *              [h_offsets[s], h_offsets[s+1])
 *   d_positions int32[n_total]  Multiverse position ids (assign_positions)
 *   d_seg_id   int32[n_total]   segment id per token in creation order (GenerationDag::segments
 *                               index; NULL to skip)
 *   d_excl     int32[n_total][max_depth][2]  per-token exclusion intervals [lo, hi) of
 *              sequence-local layout rows: mask[i][j] = j <= i and j in no interval of row i.
 *              This is the compact form of build_mask (dag.cpp:243-263); unused = (0,0).
 *   d_status   int32[n_seq] per-sequence status (MV_OK / MV_ERR_MALFORMED /
 *              MV_ERR_COUNT_MISMATCH / MV_ERR_DEPTH), written asynchronously.
 *   d_workspace / workspace_bytes from mv_visibility_workspace_size.
 */
MV_API size_t mv_visibility_workspace_size(const int64_t* h_offsets, int32_t n_seq);
MV_API mv_status mv_visibility(const int32_t* d_tokens, const int64_t* h_offsets, int32_t n_seq, int32_t max_depth,
                        int32_t* d_positions, int32_t* d_seg_id, int32_t* d_excl, int32_t* d_status,
                        void* d_workspace, size_t workspace_bytes, mv_stream_t stream);

/*
 * Teacher-forced training batch (dag::build_training_batch, dag.hpp:124-139, dag.cpp:314-359) for a
 * batch of tag streams: everything mv_visibility computes (token ids are the input; layout order is
 * stream order) plus, per token, the next-token target (-1 where the row has none: a path's last
 * token, unless its block has one path, and the sequence's last token) and the loss mask
 * (target >= 0 and, unless tag_loss, a non-tag target; BatchOptions::tag_loss, dag.hpp:120-122).
 *   d_targets int32[n_total]; d_loss_mask uint8[n_total]; same workspace as mv_visibility.
 */
MV_API mv_status mv_training_batch(const int32_t* d_tokens, const int64_t* h_offsets, int32_t n_seq, int32_t max_depth,
                                   int32_t tag_loss, int32_t* d_positions, int32_t* d_excl, int32_t* d_targets,
                                   uint8_t* d_loss_mask, int32_t* d_status, void* d_workspace, size_t workspace_bytes,
                                   mv_stream_t stream);

/*
 * Dense legacy dag::Mask (dag.hpp:59-73) from the intervals: rows [row0, row1) of one
 * sequence of length n, MSB-first packed bits, row-major ((row1-row0)*n bits).
 */
MV_API mv_status mv_mask_packed(const int32_t* d_excl, int32_t n, int32_t max_depth, int32_t row0, int32_t row1,
                         uint8_t* d_out, mv_stream_t stream);

/*
 * Prefill tile map: classifies every (q-tile, k-tile) of block size `tile` as skipped
 * (fully masked), full (no masking needed) or partial. d_count[n_qt] receives the
 * number of non-skipped k-tiles per q-tile; d_list[n_qt][n_qt] their k-tile indices
 * (ascending), with bit 30 set for partial tiles. Returns the total visible pair count
 * (popcount of the mask) in *d_visible_pairs (int64, accumulated atomically; zero it first).
 */
MV_API mv_status mv_tile_map(const int32_t* d_excl, int32_t n, int32_t max_depth, int32_t tile, int32_t* d_count,
                      int32_t* d_list, unsigned long long* d_visible_pairs, mv_stream_t stream);

/* ======================================================================== */
/* K2 — paged KV store with Process-stage fork and Reduce-stage merge        */
/* ======================================================================== */
/*
 * Replaces kv::RadixStore (kvcache.hpp:60-154). Pages of 16 token slots live in device
 * memory; each handle owns a device page table of ragged (page, begin, count) entries
 * (SURVEY.md §7 H1). fork copies page tables and bumps page refcounts; merge concatenates
 * page tables; neither moves a KV byte (bytes_copied == 0 by construction, reported
 * from a device counter of payload bytes written by fork/merge kernels).
 *
 * Slots of one page may be shared by several tables: a page is "sealed" for in-place
 * appends once its tail is shared (fork, merge, functional extend).
 */
typedef struct mv_kv_store mv_kv_store;

typedef struct {
  int32_t num_pages;      /* page pool size; tokens capacity = 16 * num_pages (CapacityExceeded beyond) */
  int32_t record_bytes;   /* opaque per-token payload record (RadixStore payload_record_size); 0 = none */
  int32_t layers;         /* attention KV planes: bf16 K and V per layer, head-major [kv_head][page][16][head_dim] */
  int32_t kv_heads;       /*   (0 = no attention plane) */
  int32_t head_dim;       /*   64 or 128 when kv_heads > 0 (the attention kernels' native head dims) */
  int64_t table_entries;  /* device page-table arena capacity in entries (0 = 4 * num_pages + 65536) */
  double rope_base;       /* rotary base for K at append (toy_model.cpp:30-41); 0 = 10000 */
} mv_kv_config;

/* StorageStats (kvcache.hpp:43-50); physical/node/refcount are page-level for this store. */
typedef struct {
  uint64_t physical_tokens_stored;   /* distinct slots referenced by live handles */
  uint64_t logical_tokens_reachable; /* sum of live handle lengths */
  uint64_t bytes_copied_on_last_op;  /* payload bytes duplicated by the last op: always 0 */
  uint64_t live_handles;
  uint64_t node_count;               /* pages with refcount > 0 */
  uint64_t total_refcount;           /* sum of page refcounts (one per table entry) */
  uint64_t free_pages;
} mv_kv_stats;

MV_API mv_status mv_kv_store_create(const mv_kv_config* cfg, mv_kv_store** out);
MV_API mv_status mv_kv_store_destroy(mv_kv_store* s);
/* All store kernels are issued on this stream (default: NULL). */
MV_API mv_status mv_kv_set_stream(mv_kv_store* s, mv_stream_t stream);
/* Device pointers of the attention planes (for callers that run their own kernels). */
MV_API mv_status mv_kv_planes(mv_kv_store* s, int32_t layer, void** d_k, void** d_v);

/* RadixStore::create (kvcache.hpp:66-67). */
MV_API mv_status mv_kv_create(mv_kv_store* s, uint64_t* out_handle);
/* RadixStore::extend (kvcache.hpp:69-75): new handle = h ++ tokens; h stays live.
 * h_payloads: n * record_bytes host bytes, or NULL. */
MV_API mv_status mv_kv_extend(mv_kv_store* s, uint64_t h, const int32_t* h_tokens, int64_t n, const void* h_payloads,
                       uint64_t* out_handle);
/* RadixStore::fork (kvcache.hpp:77-78): n handles resolving to h's tokens. */
MV_API mv_status mv_kv_fork(mv_kv_store* s, uint64_t h, int32_t n, uint64_t* out_handles);
/* RadixStore::merge (kvcache.hpp:80-83): prefix ++ each branch's suffix, in order.
 * MV_ERR_NOT_DESCENDANT if a branch is shorter or does not physically share the prefix
 * slot-for-slot (kvcache.cpp:262-275). */
MV_API mv_status mv_kv_merge(mv_kv_store* s, uint64_t prefix, const uint64_t* h_branches, int32_t n_branches,
                      uint64_t* out_handle);
/* RadixStore::release (kvcache.hpp:85-87). */
MV_API mv_status mv_kv_release(mv_kv_store* s, uint64_t h);
MV_API mv_status mv_kv_length(mv_kv_store* s, uint64_t h, int64_t* out_len);
MV_API mv_status mv_kv_stats_get(mv_kv_store* s, mv_kv_stats* out);
/* RadixStore::resolve / resolve_payloads / resolve_slots (kvcache.hpp:91-95), into host
 * buffers of length() entries (payloads: length() * record_bytes bytes). */
MV_API mv_status mv_kv_resolve(mv_kv_store* s, uint64_t h, int32_t* h_tokens);
MV_API mv_status mv_kv_resolve_payloads(mv_kv_store* s, uint64_t h, void* h_out);
MV_API mv_status mv_kv_resolve_slots(mv_kv_store* s, uint64_t h, uint32_t* h_slots);

/*
 * Engine fast path (replaces the per-token extend + release pair of engine.cpp:639-641):
 * append one token to each of n handles IN PLACE (handle ids unchanged), allocating pages
 * on device as needed, and write the token's attention K/V for `layer`:
 * K is rotated (interleaved RoPE, toy_model.cpp:30-41) at d_positions[i] before it is
 * cached; V is cached as given (toy_model.cpp:116-119).
 *   d_tokens int32[n]; d_positions int32[n]; d_k, d_v bf16[n][kv_heads][head_dim]
 * Pass d_k = d_v = NULL to append token ids only.
 */
MV_API mv_status mv_kv_append(mv_kv_store* s, const uint64_t* h_handles, int32_t n, const int32_t* d_tokens,
                       const int32_t* d_positions, int32_t layer, const void* d_k, const void* d_v);
/* Write K/V of the LAST token of each handle for another layer (multi-layer models). */
MV_API mv_status mv_kv_write_last(mv_kv_store* s, const uint64_t* h_handles, int32_t n, const int32_t* d_positions,
                           int32_t layer, const void* d_k, const void* d_v);
/* Bulk prefill of a handle's attention plane: n tokens appended in place with K/V rows
 * d_k/d_v bf16[n][kv_heads][head_dim] at positions d_positions[n]. */
MV_API mv_status mv_kv_append_many(mv_kv_store* s, uint64_t h, int64_t n, const int32_t* d_tokens,
                            const int32_t* d_positions, int32_t layer, const void* d_k, const void* d_v);
/* K/V of tokens [first, first + n) of handle h for `layer` (bf16 [n][kv_heads][head_dim], K rotated at
 * d_positions[i], or not at all when d_positions is NULL): the other layers of a bulk prefill. */
MV_API mv_status mv_kv_write_range(mv_kv_store* s, uint64_t h, int64_t first, int64_t n, const int32_t* d_positions,
                                   int32_t layer, const void* d_k, const void* d_v);
/* Gather a handle's cached K and V (post-RoPE, bf16 [len][kv_heads][head_dim]) into device buffers. */
MV_API mv_status mv_kv_gather_kv(mv_kv_store* s, uint64_t h, int32_t layer, void* d_k, void* d_v);

/* ======================================================================== */
/* K4 — branch-parallel paged decode attention (split-KV, cascade)           */
/* ======================================================================== */
/*
 * Replaces the attention core of ToyModel::step (toy_model.cpp:121-157) over the
 * context that engine.cpp:603-607 resolves for every active lane — for ALL lanes of
 * all requests in one launch. Shared Map-prefix pages (from fork lineage) are read once
 * per group of sibling branches (cascade); GQA query heads of one KV head are packed
 * into the same tile.
 *
 *   h_handles[n]   the decoding sequences (their current cache includes the new token)
 *   d_q            bf16[n][q_heads][head_dim] pre-RoPE queries; rotated in-kernel at
 *                  d_positions[i] (interleaved RoPE)
 *   d_out          [n][q_heads][head_dim], bf16 (out_dtype 0) or fp32 (out_dtype 1); the fp32
 *                  form exposes the kernel's fp32 result before the bf16 store rounding
 *                  (2^-9 |o|), which is what the 2e-3 parity contract is checked on
 * The plan (cascade units, split-KV chunks, partial buffers) is built and cached inside the
 * store; it is rebuilt automatically when the handles' page tables change.
 */
MV_API mv_status mv_attn_decode(mv_kv_store* s, int32_t layer, const uint64_t* h_handles, int32_t n, int32_t q_heads,
                         const void* d_q, const int32_t* d_positions, void* d_out, int32_t out_dtype);

/* Decode-plan statistics of the last mv_attn_decode call on this store (host ints). */
typedef struct {
  int32_t units, chunks, work_items, partial_slots;
  int64_t unique_kv_tokens;   /* tokens of KV read once per step (sum over units) */
  int64_t naive_kv_tokens;    /* tokens a per-branch decode would read (sum of lengths) */
} mv_decode_plan_info;
MV_API mv_status mv_attn_decode_plan_info(mv_kv_store* s, mv_decode_plan_info* out);
/* Measurement hook: with max_calls > 0, the next max_calls mv_attn_decode calls on this store record a CUDA
 * event pair around the decode_tc launch alone (the RoPE pre-pass and the split-KV combine outside it).
 * A call with h_n != NULL first writes the recorded launches' durations (ms) to h_ms[0..*h_n) (waiting for
 * them); every call re-arms the recording for max_calls more calls (0 = off). */
MV_API mv_status mv_attn_decode_kernel_timing(mv_kv_store* s, int32_t max_calls, float* h_ms, int32_t* h_n);

/* ======================================================================== */
/* K3 — branch-masked prefill attention (tcgen05 / TMEM / TMA)               */
/* ======================================================================== */
/*
 * Replaces the attention inside ToyModel::forward (toy_model.cpp:174-202) for a whole
 * structured sequence at once:
 *   d_q bf16[n][q_heads][128], d_k / d_v bf16[n][kv_heads][128] (pre-RoPE, rotated in
 *   kernel at d_positions), d_excl from mv_visibility, d_out [n][q_heads][128] bf16
 *   (out_dtype 0) or fp32 (out_dtype 1).
 * Fully masked cross-branch tiles are skipped using the tile map.
 */
MV_API size_t mv_prefill_workspace_size(int32_t n, int32_t q_heads, int32_t kv_heads);
MV_API mv_status mv_attn_prefill(const void* d_q, const void* d_k, const void* d_v, const int32_t* d_positions,
                          const int32_t* d_excl, int32_t max_depth, int32_t n, int32_t q_heads, int32_t kv_heads,
                          double rope_base, void* d_out, int32_t out_dtype, void* d_workspace,
                          size_t workspace_bytes, mv_stream_t stream);
/* The same with an explicit head dim (64 or 128; the two above are head_dim 128): every [..][128]
 * above reads [..][head_dim].  ToyModel's d_h = model_dim / heads (toy_model.hpp:29) is 64 at C1. */
MV_API size_t mv_prefill_workspace_size_hd(int32_t n, int32_t q_heads, int32_t kv_heads, int32_t head_dim);
MV_API mv_status mv_attn_prefill_hd(const void* d_q, const void* d_k, const void* d_v, const int32_t* d_positions,
                             const int32_t* d_excl, int32_t max_depth, int32_t n, int32_t q_heads,
                             int32_t kv_heads, int32_t head_dim, double rope_base, void* d_out, int32_t out_dtype,
                             void* d_workspace, size_t workspace_bytes, mv_stream_t stream);

/*
 * K5 — per-lane tag interpreter (replaces engine.cpp:323-415 feed_interpreter, with the BUG-2
 * fix, and the merge-completion reset at engine.cpp:793).
 * d_state: MV_INTERP_STATE_WORDS int32 per lane (opaque), set up by mv_interp_init; d_is_child
 * (nullable: all root lanes) marks worker lanes (LaneRuntime::parent >= 0).
 * mv_interp_feed walks d_events [n_steps][n_lanes] (token ids, 0..9 the tags in TagKind order;
 * MV_INTERP_IDLE: no call this step; MV_INTERP_MERGED: the lane's paths were merged) and writes
 * d_action [n_steps][n_lanes] (MV_ACT_*) and d_arg (spawn count for MV_ACT_SPAWN, MV_VIOL_* for
 * MV_ACT_VIOLATION, else 0). A violation leaves the lane state unchanged, as the reference does.
 * Optional d_spawns: (step, lane, count) triples appended in no particular order at
 * *d_n_spawns (caller-zeroed, device memory).
 */
#define MV_INTERP_STATE_WORDS 2
#define MV_INTERP_IDLE (-1)
#define MV_INTERP_MERGED (-2)
#define MV_ACT_NONE 0
#define MV_ACT_SPAWN 1
#define MV_ACT_WORKER_DONE 2
#define MV_ACT_VIOLATION 3
#define MV_VIOL_PATH_CLOSE_OUTSIDE 1          /* "</Path> outside any path" */
#define MV_VIOL_UNEXPECTED_SEQUENTIAL 2       /* "unexpected <tag> in sequential decode" */
#define MV_VIOL_EXPECTED_GOAL 3               /* "expected <Goal> after <Parallel>" */
#define MV_VIOL_TEXT_BETWEEN_OUTLINES 4       /* "text between outlines" */
#define MV_VIOL_NESTED_OUTLINE 5              /* "nested <Outline>" */
#define MV_VIOL_OUTLINE_CLOSE_WITHOUT_OPEN 6  /* "</Outline> without <Outline>" */
#define MV_VIOL_GOAL_CLOSE_IN_OUTLINE 7       /* "</Goal> inside <Outline>" */
#define MV_VIOL_ZERO_OUTLINES 8               /* "</Goal> with zero outlines" */
#define MV_VIOL_UNEXPECTED_IN_GOAL 9          /* "unexpected <tag> inside <Goal>" */
#define MV_VIOL_WAITING 10                    /* "token while waiting for paths" */
#define MV_VIOL_EXPECTED_CONCLUSION 11        /* "expected <Conclusion> after merge" */
#define MV_VIOL_UNEXPECTED_IN_CONCLUSION 12   /* "unexpected <tag> inside <Conclusion>" */
#define MV_VIOL_EXPECTED_PARALLEL_CLOSE 13    /* "expected </Parallel> after </Conclusion>" */
#define MV_VIOL_MERGE_NO_BLOCK 14             /* merge with no open block (undefined in the reference) */
MV_API mv_status mv_interp_init(int32_t* d_state, int32_t n_lanes, const int32_t* d_is_child, mv_stream_t stream);
MV_API mv_status mv_interp_feed(int32_t* d_state, int32_t n_lanes, const int32_t* d_events, int32_t n_steps,
                                int32_t* d_action, int32_t* d_arg, int32_t* d_spawns, int32_t* d_n_spawns,
                                mv_stream_t stream);

/* ======================================================================== */
/* The reference's toy transformer on the device      */
/* ======================================================================== */
/*
 * toy::ToyModel (toy_model.hpp:71-92, toy_model.cpp:45-221) with every layer op on the GPU: fp32
 * projections / tanh MLP / unembed, fp64 RoPE at the token's position, attention through K4 / K3.
 * Head dims below 128 ride the 128-wide attention kernels zero-padded.
 * Weights: host fp64 in ToyModelWeights order (toy_model.cpp:58-68): embedding [V][D]; per layer
 * wq, wk, wv, wo [D][D], w_up [4D][D], w_down [D][4D]; unembed [V][D]; mv_toy_weight_count doubles.
 */
typedef struct mv_toy mv_toy;
typedef struct {
  int32_t layers, heads, model_dim, vocab;
  double rope_base; /* 0 = 10000 */
} mv_toy_config;
MV_API size_t mv_toy_weight_count(const mv_toy_config* cfg);
MV_API mv_status mv_toy_create(const mv_toy_config* cfg, const double* h_weights, mv_toy** out);
MV_API mv_status mv_toy_destroy(mv_toy* m);
/* The attention kernels' head dim for a model head dim: d_h itself when it is 64 or 128 (native
 * kernels), else 128 (q / k / v zero-padded, q pre-scaled by sqrt(128 / d_h)).  Toy stores use it. */
MV_API int32_t mv_attn_head_dim(int32_t model_head_dim);
/*
 * ToyModel::step for n lanes at once (engine.cpp:603-641 batched): each lane's token joins its cache
 * (K/V of every layer appended in place into `s`, whose planes must be layers x heads x
 * mv_attn_head_dim(model_dim / heads)) and
 * attends over it.  d_tokens / d_positions int32[n]; d_logits fp32 [n][V]; optional d_hidden fp32
 * [n][D] and d_kv fp32 [n][2 * layers * D] (the reference's cache record: per layer rotated K | V).
 * Runs on the store's stream.
 */
MV_API mv_status mv_toy_step(mv_toy* m, mv_kv_store* s, const uint64_t* h_handles, int32_t n, const int32_t* d_tokens,
                             const int32_t* d_positions, float* d_logits, float* d_hidden, float* d_kv);
/* Appends ctx_len tokens to handle h from the reference's host cache records (fp64 [ctx_len][2 * layers *
 * D]; resolve_payloads of engine.cpp:603): the legacy ToyModel::step(context_kv, ...) entry point. */
MV_API mv_status mv_toy_load_context(mv_toy* m, mv_kv_store* s, uint64_t h, const double* h_records, int64_t ctx_len);
/* ToyModel::forward (toy_model.cpp:174-202) over one structured sequence: d_positions / d_excl from
 * mv_visibility (or mv_training_batch); d_logits fp32 [n][V]; optional d_hidden fp32 [n][D]. */
MV_API mv_status mv_toy_forward(mv_toy* m, const int32_t* d_tokens, int32_t n, const int32_t* d_positions,
                                const int32_t* d_excl, int32_t max_depth, float* d_logits, float* d_hidden,
                                mv_stream_t stream);
MV_API mv_status mv_toy_get_config(const mv_toy* m, mv_toy_config* out);
MV_API int32_t mv_toy_vocab(const mv_toy* m);
/* Greedy sampling (engine.cpp:543-556): the first index of each row's maximum. */
MV_API mv_status mv_argmax_rows(const float* d_x, int32_t n, int32_t cols, int32_t* d_idx, mv_stream_t stream);

/* ======================================================================== */
/* Engine: the batched Multiverse decode loop  */
/* ======================================================================== */
/*
 * engine::run_forced / run_free (engine.cpp:928-950) over the device hot path: per step ONE batched
 * device pass for every active lane (mv_toy_step: KV append + K4 decode + layer algebra; greedy argmax;
 * K5 mv_interp_feed for the tag interpreter of every lane); the host reads back the interpreter actions
 * and sampled ids (one small copy per step) and spawns (mv_kv_fork + injected <Path>, label), retires
 * (</Path> -> zombie) and merges (zero-copy mv_kv_merge + injected <Conclusion>) as the reference's
 * Simulator does (engine.cpp:498-802).  Positions are runtime state (engine.cpp:705, :788).
 */
typedef struct {
  int32_t max_worker_tokens;   /* EngineLimits (engine.hpp:64-67); 0 = 4096 */
  int32_t max_request_tokens;  /* 0 = 4096 */
  int32_t num_pages;           /* paged-store pages for the run; 0 = 4096 */
} mv_engine_options;
#define MV_ENGINE_FAIL_NONE 0
#define MV_ENGINE_FAIL_GRAMMAR 1 /* FailureKind::GrammarViolationDuringDecode */
#define MV_ENGINE_FAIL_LIMIT 2   /* FailureKind::LimitExceeded */
typedef struct {
  int32_t status;               /* RunStatus: 0 Done, 1 Failed */
  int32_t failure;              /* MV_ENGINE_FAIL_* */
  char failure_detail[256];     /* SimulationReport::failure_detail */
  int64_t steps, total_tokens, merges, spawns, lanes, events;
} mv_engine_report;
/* SimEvent (engine.hpp:85-97): step, lane, kind (EventKind order), token id or spawn count, source index */
#define MV_EVT_DECODE 0
#define MV_EVT_PREFILL 1
#define MV_EVT_SPAWN 2
#define MV_EVT_ZOMBIE 3
#define MV_EVT_MERGE 4
#define MV_EVT_DONE 6
#define MV_EVT_FAILED 7
typedef struct {
  int64_t step;
  int32_t request, lane, kind, token, source;  /* lane: index within its request */
} mv_engine_event;
/* Token id of a path index label ("1:", "2.1:", ...; tok::Tokenizer::text_token, engine.cpp:711-715). */
typedef int32_t (*mv_engine_label_fn)(void* ctx, const char* label);
/* Forced run (run_forced with record_logits): h_tokens is the tag stream; h_logits fp32 [n][vocab] by
 * source index (NULL to skip); events into h_events[events_cap] (report.events counts them all). */
MV_API mv_status mv_engine_run_forced(mv_toy* m, const int32_t* h_tokens, int32_t n, const mv_engine_options* opt,
                                      mv_stream_t stream, float* h_logits, mv_engine_event* h_events,
                                      int64_t events_cap, mv_engine_report* report);
/* A batch of forced requests in one engine (run_batch, engine.cpp:952-966, with the toy model attached):
 * stream r is h_tokens[h_offsets[r], h_offsets[r+1]); every step is ONE device pass over the active
 * lanes of ALL requests; h_logits fp32 [h_offsets[n_req]][vocab] by flat source index; the report
 * carries the first failed request's kind and detail (finalize, engine.cpp:835-880). */
MV_API mv_status mv_engine_run_batch(mv_toy* m, const int32_t* h_tokens, const int64_t* h_offsets, int32_t n_req,
                                     const mv_engine_options* opt, mv_stream_t stream, float* h_logits,
                                     mv_engine_event* h_events, int64_t events_cap, mv_engine_report* report);
/* Greedy free-running decode after an injected prompt (run_free); stops after max_steps (0: none). */
MV_API mv_status mv_engine_run_free(mv_toy* m, const int32_t* h_prompt, int32_t n_prompt, int32_t max_steps,
                                    const mv_engine_options* opt, mv_engine_label_fn label_fn, void* label_ctx,
                                    mv_stream_t stream, mv_engine_event* h_events, int64_t events_cap,
                                    mv_engine_report* report);

#ifdef __cplusplus
}
#endif

#endif /* MULTIVERSE_B200_H_ */
