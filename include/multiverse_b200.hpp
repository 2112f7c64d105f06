// multiverse_b200.hpp — C++20 host shim over the C-ABI (multiverse_b200.h).
//
// Mirrors the reference's proj/core hot-path interface so its callers (engine.cpp,
// tests) can switch by changing the namespace:
//   multiverse::kv::RadixStore / CacheError / StorageStats / SequenceHandle  (kvcache.hpp:32-101)
//   multiverse::dag::build_visibility / VisibilitySpec / Mask                 (dag.hpp:59-110)
//   the attention core of multiverse::toy::ToyModel::step / forward           (toy_model.cpp:121-202)
// Same method names, argument meaning and exception kinds; values live on the device.
// Header-only; link with -lmvb200 -lcudart.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "multiverse_b200.h"

namespace multiverse_b200 {

class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace grammar {
// grammar::ParseError (grammar.hpp:136-152)
class ParseError : public std::runtime_error {
 public:
  enum class Kind { MalformedStructure, CountMismatch };
  ParseError(Kind kind, const std::string& what) : std::runtime_error(what), kind_(kind) {}
  Kind kind() const { return kind_; }

 private:
  Kind kind_;
};
}  // namespace grammar

namespace kv {

using TokenId = std::int32_t;

// kv::CacheError (kvcache.hpp:32-41)
class CacheError : public std::runtime_error {
 public:
  enum class Kind { UnknownHandle, DoubleRelease, CapacityExceeded, BranchNotDescendant };
  CacheError(Kind kind, const std::string& what) : std::runtime_error(what), kind_(kind) {}
  Kind kind() const { return kind_; }

 private:
  Kind kind_;
};

}  // namespace kv

// Maps a C-ABI status to the reference's exception types (kvcache.hpp:32-41,
// grammar.hpp:136-152, std::invalid_argument).
inline void check(mv_status st) {
  if (st == MV_OK) return;
  const std::string msg = mv_last_error();
  switch (st) {
    case MV_ERR_UNKNOWN_HANDLE: throw kv::CacheError(kv::CacheError::Kind::UnknownHandle, msg);
    case MV_ERR_DOUBLE_RELEASE: throw kv::CacheError(kv::CacheError::Kind::DoubleRelease, msg);
    case MV_ERR_CAPACITY: throw kv::CacheError(kv::CacheError::Kind::CapacityExceeded, msg);
    case MV_ERR_NOT_DESCENDANT: throw kv::CacheError(kv::CacheError::Kind::BranchNotDescendant, msg);
    case MV_ERR_MALFORMED: throw grammar::ParseError(grammar::ParseError::Kind::MalformedStructure, msg);
    case MV_ERR_COUNT_MISMATCH: throw grammar::ParseError(grammar::ParseError::Kind::CountMismatch, msg);
    case MV_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    default: throw CudaError(msg);
  }
}

inline void cuda_check(cudaError_t e) {
  if (e != cudaSuccess) throw CudaError(cudaGetErrorString(e));
}

// Minimal owning device buffer.
template <typename T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t n) : n_(n) {
    if (n) cuda_check(cudaMalloc(&p_, n * sizeof(T)));
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr, o.n_ = 0; }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    return *this;
  }
  ~DeviceBuffer() { cudaFree(p_); }
  T* data() const { return p_; }
  std::size_t size() const { return n_; }
  void upload(const T* h, std::size_t n) { cuda_check(cudaMemcpy(p_, h, n * sizeof(T), cudaMemcpyHostToDevice)); }
  std::vector<T> download() const {
    std::vector<T> h(n_);
    if (n_) cuda_check(cudaMemcpy(h.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost));
    return h;
  }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

namespace kv {

// kv::StorageStats (kvcache.hpp:43-50). node_count / total_refcount are page-level here.
struct StorageStats {
  std::size_t physical_tokens_stored = 0;
  std::size_t logical_tokens_reachable = 0;
  std::size_t bytes_copied_on_last_op = 0;
  std::size_t live_handles = 0;
  std::size_t node_count = 0;
  std::size_t total_refcount = 0;
};

// kv::SequenceHandle (kvcache.hpp:52-58)
struct SequenceHandle {
  std::uint64_t id = 0;
  std::size_t length = 0;
  bool valid() const { return id != 0; }
};

// kv::RadixStore (kvcache.hpp:60-101) on the device page store. capacity_tokens is
// rounded up to whole 16-token pages. The attention plane (layers x kv_heads x 128 bf16
// K and V per token) is optional: kv_heads = 0 gives the payload-only store the
// reference's engine uses in scripted mode (engine.cpp:444-449).
class RadixStore {
 public:
  explicit RadixStore(std::size_t payload_record_size = 0, std::size_t capacity_tokens = 1u << 20, int layers = 0,
                      int kv_heads = 0, double rope_base = 10000.0)
      : record_size_(payload_record_size) {
    mv_kv_config cfg{};
    cfg.num_pages = static_cast<int32_t>((capacity_tokens + 15) / 16);
    cfg.record_bytes = static_cast<int32_t>(payload_record_size);
    cfg.layers = kv_heads > 0 ? layers : 0;
    cfg.kv_heads = kv_heads;
    cfg.head_dim = 128;
    cfg.rope_base = rope_base;
    check(mv_kv_store_create(&cfg, &s_));
  }
  RadixStore(const RadixStore&) = delete;
  RadixStore& operator=(const RadixStore&) = delete;
  ~RadixStore() { mv_kv_store_destroy(s_); }

  std::size_t record_size() const { return record_size_; }
  mv_kv_store* native() const { return s_; }
  void set_stream(cudaStream_t st) { check(mv_kv_set_stream(s_, st)); }

  SequenceHandle create() {
    SequenceHandle h;
    check(mv_kv_create(s_, &h.id));
    return h;
  }

  SequenceHandle extend(const SequenceHandle& h, std::span<const TokenId> tokens,
                        std::span<const std::byte> payloads = {}) {
    // same check as kvcache.cpp:153-156 (empty payloads are accepted and stored as zeros)
    if (record_size_ > 0 && !payloads.empty() && payloads.size() != tokens.size() * record_size_)
      throw std::invalid_argument("payload byte count does not match token count");
    SequenceHandle out;
    check(mv_kv_extend(s_, h.id, tokens.data(), static_cast<int64_t>(tokens.size()),
                       payloads.empty() ? nullptr : payloads.data(), &out.id));
    out.length = length_of(out.id);
    return out;
  }

  std::vector<SequenceHandle> fork(const SequenceHandle& h, int n) {
    if (n < 0) throw std::invalid_argument("fork count must be >= 0");
    std::vector<std::uint64_t> ids(static_cast<std::size_t>(n));
    check(mv_kv_fork(s_, h.id, n, ids.data()));
    const std::size_t len = length_of(h.id);
    std::vector<SequenceHandle> out;
    out.reserve(ids.size());
    for (auto id : ids) out.push_back({id, len});
    return out;
  }

  SequenceHandle merge(const SequenceHandle& prefix, std::span<const SequenceHandle> branches) {
    std::vector<std::uint64_t> ids;
    ids.reserve(branches.size());
    for (const auto& b : branches) ids.push_back(b.id);
    SequenceHandle out;
    check(mv_kv_merge(s_, prefix.id, ids.data(), static_cast<int32_t>(ids.size()), &out.id));
    out.length = length_of(out.id);
    return out;
  }

  void release(const SequenceHandle& h) { check(mv_kv_release(s_, h.id)); }

  StorageStats stats() const {
    mv_kv_stats st{};
    check(mv_kv_stats_get(s_, &st));
    return {st.physical_tokens_stored, st.logical_tokens_reachable, st.bytes_copied_on_last_op,
            st.live_handles,           st.node_count,               st.total_refcount};
  }

  std::vector<TokenId> resolve(const SequenceHandle& h) const {
    std::vector<TokenId> out(length_of(h.id));
    check(mv_kv_resolve(s_, h.id, out.data()));
    return out;
  }
  std::vector<std::byte> resolve_payloads(const SequenceHandle& h) const {
    std::vector<std::byte> out(length_of(h.id) * record_size_);
    check(mv_kv_resolve_payloads(s_, h.id, out.data()));
    return out;
  }
  std::vector<std::uint32_t> resolve_slots(const SequenceHandle& h) const {
    std::vector<std::uint32_t> out(length_of(h.id));
    check(mv_kv_resolve_slots(s_, h.id, out.data()));
    return out;
  }

  // Engine fast path (engine.cpp:639-641 extend + release of the old handle, in place):
  // append one token per handle with its attention K/V (device bf16 [n][kv_heads][128]).
  void append(std::span<const std::uint64_t> handles, const int32_t* d_tokens, const int32_t* d_positions, int layer,
              const void* d_k, const void* d_v) {
    check(mv_kv_append(s_, handles.data(), static_cast<int32_t>(handles.size()), d_tokens, d_positions, layer, d_k,
                       d_v));
  }

 private:
  std::size_t length_of(std::uint64_t id) const {
    int64_t n = 0;
    check(mv_kv_length(s_, id, &n));
    return static_cast<std::size_t>(n);
  }

  mv_kv_store* s_ = nullptr;
  std::size_t record_size_ = 0;
};

}  // namespace kv

namespace dag {

// dag::Mask (dag.hpp:59-73), dense, materialised from the device intervals.
class Mask {
 public:
  Mask() = default;
  explicit Mask(std::size_t n) : n_(n), bits_(n * n, 0) {}
  std::size_t size() const { return n_; }
  bool at(std::size_t i, std::size_t j) const { return bits_[i * n_ + j] != 0; }
  void set(std::size_t i, std::size_t j, bool v) { bits_[i * n_ + j] = v ? 1 : 0; }
  bool operator==(const Mask&) const = default;

 private:
  std::size_t n_ = 0;
  std::vector<std::uint8_t> bits_;
};

// dag::VisibilitySpec (dag.hpp:104-110) plus the compact device form the kernels use.
struct VisibilitySpec {
  std::vector<int> positions;
  Mask mask;
};

struct DeviceVisibility {
  int n = 0, max_depth = 0;
  DeviceBuffer<int32_t> positions;  // int32[n]
  DeviceBuffer<int32_t> seg_id;     // int32[n]
  DeviceBuffer<int32_t> excl;       // int32[n][max_depth][2]
};

// Tag-stream token ids (tok::Tokenizer ids, tokenizer.cpp:56-63) -> device positions and
// exclusion intervals. Throws grammar::ParseError like grammar::parse (grammar.cpp:156-294).
inline DeviceVisibility build_visibility_device(std::span<const int32_t> tokens, int max_depth = 4,
                                                cudaStream_t stream = nullptr) {
  DeviceVisibility v;
  v.n = static_cast<int>(tokens.size());
  v.max_depth = max_depth;
  const std::size_t n = std::max<std::size_t>(tokens.size(), 1);
  DeviceBuffer<int32_t> d_tok(n);
  if (!tokens.empty()) d_tok.upload(tokens.data(), tokens.size());
  v.positions = DeviceBuffer<int32_t>(n);
  v.seg_id = DeviceBuffer<int32_t>(n);
  v.excl = DeviceBuffer<int32_t>(n * static_cast<std::size_t>(max_depth) * 2);
  DeviceBuffer<int32_t> status(1);
  const int64_t offs[2] = {0, static_cast<int64_t>(tokens.size())};
  const std::size_t ws_bytes = mv_visibility_workspace_size(offs, 1);
  DeviceBuffer<std::uint8_t> ws(std::max<std::size_t>(ws_bytes, 1));
  check(mv_visibility(d_tok.data(), offs, 1, max_depth, v.positions.data(), v.seg_id.data(), v.excl.data(),
                      status.data(), ws.data(), ws_bytes, stream));
  cuda_check(cudaStreamSynchronize(stream));
  const auto st = static_cast<mv_status>(status.download()[0]);
  if (st == MV_ERR_DEPTH && max_depth < 64)  // deeper nesting than interval slots: grow the capacity
    return build_visibility_device(tokens, std::min(2 * max_depth, 64), stream);
  check(st);
  return v;
}

// dag::build_visibility (dag.hpp:104-110): host positions + dense mask.
inline VisibilitySpec build_visibility(std::span<const int32_t> tokens, int max_depth = 4) {
  DeviceVisibility v = build_visibility_device(tokens, max_depth);
  VisibilitySpec out;
  const std::size_t n = tokens.size();
  out.mask = Mask(n);
  if (n == 0) return out;
  auto pos = v.positions.download();
  out.positions.assign(pos.begin(), pos.begin() + static_cast<std::ptrdiff_t>(n));
  DeviceBuffer<std::uint8_t> bits((n * n + 7) / 8);
  check(mv_mask_packed(v.excl.data(), v.n, max_depth, 0, v.n, bits.data(), nullptr));
  auto h = bits.download();
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < n; ++j) {
      const std::size_t b = i * n + j;
      out.mask.set(i, j, (h[b >> 3] >> (7 - (b & 7))) & 1);
    }
  return out;
}

}  // namespace dag

namespace attn {

// Attention core of ToyModel::step (toy_model.cpp:121-157) for every lane in one launch:
// q bf16 [n][q_heads][128] (pre-RoPE, rotated at d_positions), out bf16 or fp32.
inline void decode(kv::RadixStore& store, int layer, std::span<const std::uint64_t> handles, int q_heads,
                   const void* d_q, const int32_t* d_positions, void* d_out, bool out_f32 = false) {
  check(mv_attn_decode(store.native(), layer, handles.data(), static_cast<int32_t>(handles.size()), q_heads, d_q,
                       d_positions, d_out, out_f32 ? 1 : 0));
}

// Attention inside ToyModel::forward (toy_model.cpp:174-202) for a whole structured sequence.
inline void prefill(const void* d_q, const void* d_k, const void* d_v, const dag::DeviceVisibility& vis, int q_heads,
                    int kv_heads, void* d_out, bool out_f32 = false, double rope_base = 10000.0,
                    cudaStream_t stream = nullptr) {
  const std::size_t ws_bytes = mv_prefill_workspace_size(vis.n, q_heads, kv_heads);
  DeviceBuffer<std::uint8_t> ws(std::max<std::size_t>(ws_bytes, 1));
  check(mv_attn_prefill(d_q, d_k, d_v, vis.positions.data(), vis.excl.data(), vis.max_depth, vis.n, q_heads, kv_heads,
                        rope_base, d_out, out_f32 ? 1 : 0, ws.data(), ws_bytes, stream));
}

}  // namespace attn

namespace dag {

// dag::build_visibility(GenerationDag&) (dag.hpp:108, dag.cpp:265-270): any GenerationDag-shaped type
// (token_layout() -> (segment id, offset) rows, segments[sid].tokens[off].id) is flattened to its
// layout-order token ids and built on the device.
template <class GenerationDag>
  requires requires(GenerationDag& g) {
    g.token_layout();
    g.segments;
  }
VisibilitySpec build_visibility(GenerationDag& g, int max_depth = 8) {
  std::vector<int32_t> ids;
  for (auto [sid, off] : g.token_layout())
    ids.push_back(g.segments[static_cast<std::size_t>(sid)].tokens[static_cast<std::size_t>(off)].id);
  return build_visibility(std::span<const int32_t>(ids), max_depth);
}

}  // namespace dag

namespace toy {

// toy::ToyModelConfig (toy_model.hpp:24-37)
struct ToyModelConfig {
  int layers = 2;
  int heads = 2;
  int model_dim = 32;
  int vocab_size = 256;
  std::uint64_t seed = 0;
  double init_range = 0.05;
  double rope_base = 10000.0;

  int head_dim() const { return model_dim / heads; }
  int hidden_dim() const { return 4 * model_dim; }
  int kv_doubles_per_token() const { return 2 * layers * model_dim; }
};

// toy::ToyModelWeights (toy_model.hpp:39-57).  init() draws the reference's weights: synth::Rng over
// std::mt19937_64 (fully specified by the C++ standard) with next_symmetric's mapping (synth.cpp:24-29),
// in the fill order of toy_model.cpp:58-68.
struct ToyModelWeights {
  ToyModelConfig config;
  struct Layer {
    std::vector<double> wq, wk, wv, wo, w_up, w_down;
  };
  std::vector<double> embedding;
  std::vector<Layer> layers;
  std::vector<double> unembed;

  static ToyModelWeights init(const ToyModelConfig& config) {
    if (config.layers < 1 || config.heads < 1 || config.model_dim < 1 || config.vocab_size < 1)
      throw std::invalid_argument("toy model dims must be >= 1");
    if (config.model_dim % config.heads != 0 || config.head_dim() % 2 != 0)
      throw std::invalid_argument("model_dim must split into even-sized heads");
    ToyModelWeights w;
    w.config = config;
    std::mt19937_64 rng(config.seed);
    auto fill = [&](std::vector<double>& v, std::size_t n) {
      v.resize(n);
      for (auto& x : v) x = (static_cast<double>(rng() >> 11) * 0x1.0p-53 * 2.0 - 1.0) * config.init_range;
    };
    const std::size_t d = static_cast<std::size_t>(config.model_dim), hid = static_cast<std::size_t>(config.hidden_dim()),
                      vocab = static_cast<std::size_t>(config.vocab_size);
    fill(w.embedding, vocab * d);
    w.layers.resize(static_cast<std::size_t>(config.layers));
    for (auto& l : w.layers) {
      fill(l.wq, d * d);
      fill(l.wk, d * d);
      fill(l.wv, d * d);
      fill(l.wo, d * d);
      fill(l.w_up, hid * d);
      fill(l.w_down, d * hid);
    }
    fill(w.unembed, vocab * d);
    return w;
  }
};

// toy::StepOutput / ForwardResult (toy_model.hpp:59-69)
struct StepOutput {
  std::vector<double> logits;
  std::vector<double> hidden;
  std::vector<double> kv;
};
struct ForwardResult {
  std::vector<double> logits;
  std::vector<double> hidden;
  std::size_t rows = 0;
  std::span<const double> logits_row(std::size_t i) const {
    const std::size_t v = logits.size() / rows;
    return {logits.data() + i * v, v};
  }
  std::span<const double> hidden_row(std::size_t i) const {
    const std::size_t d = hidden.size() / rows;
    return {hidden.data() + i * d, d};
  }
};

// toy::ToyModel (toy_model.hpp:71-92) on the device (mv_toy_*).  step() is the reference's legacy
// entry point: the caller's host context records (resolve_payloads, engine.cpp:603-607) are staged into
// a scratch handle of a device store, then ONE batched device step runs the whole layer stack with K4
// for the attention; forward() is K1 + K3 over the batch's token stream.  Both are parity paths; the
// fast path is mv_toy_step over the engine's own store (mv_engine_*).
class ToyModel {
 public:
  explicit ToyModel(const ToyModelConfig& config) : ToyModel(ToyModelWeights::init(config)) {}
  explicit ToyModel(ToyModelWeights weights) : weights_(std::move(weights)) {
    const auto& c = weights_.config;
    mv_toy_config tc{c.layers, c.heads, c.model_dim, c.vocab_size, c.rope_base};
    std::vector<double> flat;
    auto put = [&](const std::vector<double>& v) { flat.insert(flat.end(), v.begin(), v.end()); };
    put(weights_.embedding);
    for (const auto& l : weights_.layers) {
      put(l.wq);
      put(l.wk);
      put(l.wv);
      put(l.wo);
      put(l.w_up);
      put(l.w_down);
    }
    put(weights_.unembed);
    check(mv_toy_create(&tc, flat.data(), &m_));
  }
  ToyModel(const ToyModel&) = delete;
  ToyModel& operator=(const ToyModel&) = delete;
  ~ToyModel() {
    if (scratch_) mv_kv_store_destroy(scratch_);
    mv_toy_destroy(m_);
  }

  const ToyModelConfig& config() const { return weights_.config; }
  const ToyModelWeights& weights() const { return weights_; }
  mv_toy* native() const { return m_; }

  StepOutput step(std::span<const double> context_kv, std::size_t ctx_len, int token_id, int position) const {
    const auto& c = weights_.config;
    const std::size_t rec = static_cast<std::size_t>(c.kv_doubles_per_token());
    if (context_kv.size() < ctx_len * rec) throw std::invalid_argument("context kv shorter than ctx_len records");
    ensure_scratch(ctx_len + 1);
    std::uint64_t h = 0;
    check(mv_kv_create(scratch_, &h));
    check(mv_toy_load_context(m_, scratch_, h, context_kv.data(), static_cast<int64_t>(ctx_len)));
    const int32_t io[2] = {token_id, position};
    DeviceBuffer<int32_t> d_io(2);
    d_io.upload(io, 2);
    DeviceBuffer<float> logits(static_cast<std::size_t>(c.vocab_size)), hidden(static_cast<std::size_t>(c.model_dim)),
        kv(rec);
    check(mv_toy_step(m_, scratch_, &h, 1, d_io.data(), d_io.data() + 1, logits.data(), hidden.data(), kv.data()));
    StepOutput out;
    auto to64 = [](const std::vector<float>& v) { return std::vector<double>(v.begin(), v.end()); };
    out.logits = to64(logits.download());
    out.hidden = to64(hidden.download());
    out.kv = to64(kv.download());
    check(mv_kv_release(scratch_, h));
    return out;
  }

  // ToyModel::forward (toy_model.cpp:174-202) over a TrainingBatch-shaped batch (token_ids, positions,
  // mask): the visibility is rebuilt on the device from the token ids (the mask is a function of the
  // tag stream, dag.cpp:314-359).
  template <class Batch>
  ForwardResult forward(const Batch& batch) const {
    const auto& c = weights_.config;
    const std::size_t n = batch.token_ids.size();
    if (batch.mask.size() != n || batch.positions.size() != n)
      throw std::invalid_argument("batch mask/positions do not match token count");
    ForwardResult r;
    r.rows = n;
    if (n == 0) return r;
    std::vector<int32_t> ids(batch.token_ids.begin(), batch.token_ids.end());
    auto vis = dag::build_visibility_device(std::span<const int32_t>(ids), 8);
    DeviceBuffer<int32_t> d_tok(n);
    d_tok.upload(ids.data(), n);
    DeviceBuffer<float> logits(n * static_cast<std::size_t>(c.vocab_size)), hidden(n * static_cast<std::size_t>(c.model_dim));
    check(mv_toy_forward(m_, d_tok.data(), static_cast<int32_t>(n), vis.positions.data(), vis.excl.data(), vis.max_depth,
                         logits.data(), hidden.data(), nullptr));
    auto lg = logits.download();
    auto hd = hidden.download();
    r.logits.assign(lg.begin(), lg.end());
    r.hidden.assign(hd.begin(), hd.end());
    return r;
  }

  // ToyModel::loss (toy_model.cpp:204-221): mean negative log-likelihood over loss-masked targets
  template <class Batch>
  double loss(const Batch& batch) const {
    ForwardResult fwd = forward(batch);
    const std::size_t vocab = static_cast<std::size_t>(weights_.config.vocab_size);
    double total = 0.0;
    std::size_t count = 0;
    for (std::size_t i = 0; i < batch.token_ids.size(); ++i) {
      if (batch.target_ids[i] < 0 || !batch.loss_mask[i]) continue;
      auto row = fwd.logits_row(i);
      double mx = -std::numeric_limits<double>::infinity();
      for (double z : row) mx = std::max(mx, z);
      double den = 0.0;
      for (double z : row) den += std::exp(z - mx);
      total += -(row[static_cast<std::size_t>(batch.target_ids[i]) % vocab] - mx - std::log(den));
      ++count;
    }
    return count ? total / static_cast<double>(count) : 0.0;
  }

 private:
  void ensure_scratch(std::size_t tokens) const {
    const std::size_t pages = (tokens + 15) / 16 + 4;
    if (scratch_ && pages <= scratch_pages_) return;
    if (scratch_) mv_kv_store_destroy(scratch_);
    scratch_pages_ = std::max<std::size_t>(pages * 2, 256);
    mv_kv_config kc{};
    kc.num_pages = static_cast<int32_t>(scratch_pages_);
    kc.layers = weights_.config.layers;
    kc.kv_heads = weights_.config.heads;
    kc.head_dim = mv_attn_head_dim(weights_.config.head_dim());
    kc.rope_base = weights_.config.rope_base;
    check(mv_kv_store_create(&kc, &scratch_));
  }

  ToyModelWeights weights_;
  mv_toy* m_ = nullptr;
  mutable mv_kv_store* scratch_ = nullptr;  // single-writer: the reference's ToyModel is shared read-only
  mutable std::size_t scratch_pages_ = 0;
};

}  // namespace toy

}  // namespace multiverse_b200
