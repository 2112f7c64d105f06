// engine.cu — the Multiverse engine's decode loop over the device hot path (SURVEY.md §8a A11,
// §8f ranks 1 and 3).
//
// Reference behaviour replaced: engine::Simulator (engine.cpp:419-815) as run_forced / run_free
// drive it (engine.cpp:928-950): per step every active lane emits one token (an injected one, its
// script's next, or the greedy argmax of its last logits); emit (engine.cpp:599-677) computes the
// lane's logits over its cached context, extends its KV and feeds the tag interpreter, whose actions
// spawn children (fork + injected <Path> and label, :679-725), retire workers (</Path> -> zombie,
// :744-748) or fail the request; at the end of the step every waiting lane whose children are all
// zombies merges them (zero-copy, :767-802) and resumes with an injected <Conclusion>.
//
// B200 form: the reference walks lanes one by one and copies each lane's whole context out of the
// store for every token (engine.cpp:503-512, :603-605).  Here one step is ONE batched device pass for
// every active lane of every request: mv_toy_step (token append into the paged store + K4 decode
// attention + the layer algebra), the greedy argmax and K5 (mv_interp_feed: the tag interpreter of all
// lanes) run back to back on the store's stream; the host reads back one small block per step (K5
// actions and the sampled ids: the tokens a serving engine streams out anyway) and performs the
// control decisions, whose device effects (fork page tables, zero-copy merges) are kernels again.
// Positions are runtime bookkeeping as in the reference: a child starts at its parent's next position
// (:705), a merged parent continues at the maximum over its children (:788).
//
// Deliberate deviation: scripted child lanes activated by a spawn start on the NEXT step (the
// reference's comment at engine.cpp:505 states this; its loop lets pre-compiled children run in the
// spawning step, SURVEY.md §0 "minor deviation").  Tokens, positions, contexts and logits are
// unaffected; only the step count (wall units) differs on forced runs.
#include <algorithm>
#include <cstring>
#include <deque>
#include <string>
#include <vector>

#include "store.hpp"

namespace mv {
namespace {

constexpr int kTagCount_ = 10;
const char* kTagText[kTagCount_] = {"<Parallel>", "</Parallel>", "<Goal>", "</Goal>", "<Outline>",
                                    "</Outline>", "<Path>", "</Path>", "<Conclusion>", "</Conclusion>"};

// MV_VIOL_* -> InterpAction::detail (engine.cpp:323-415); {tag} is the offending token's literal
std::string violation_text(int code, int token) {
  const std::string tag = token >= 0 && token < kTagCount_ ? kTagText[token] : "w" + std::to_string(token);
  switch (code) {
    case MV_VIOL_PATH_CLOSE_OUTSIDE: return "</Path> outside any path";
    case MV_VIOL_UNEXPECTED_SEQUENTIAL: return "unexpected " + tag + " in sequential decode";
    case MV_VIOL_EXPECTED_GOAL: return "expected <Goal> after <Parallel>";
    case MV_VIOL_TEXT_BETWEEN_OUTLINES: return "text between outlines";
    case MV_VIOL_NESTED_OUTLINE: return "nested <Outline>";
    case MV_VIOL_OUTLINE_CLOSE_WITHOUT_OPEN: return "</Outline> without <Outline>";
    case MV_VIOL_GOAL_CLOSE_IN_OUTLINE: return "</Goal> inside <Outline>";
    case MV_VIOL_ZERO_OUTLINES: return "</Goal> with zero outlines";
    case MV_VIOL_UNEXPECTED_IN_GOAL: return "unexpected " + tag + " inside <Goal>";
    case MV_VIOL_WAITING: return "token while waiting for paths";
    case MV_VIOL_EXPECTED_CONCLUSION: return "expected <Conclusion> after merge";
    case MV_VIOL_UNEXPECTED_IN_CONCLUSION: return "unexpected " + tag + " inside <Conclusion>";
    case MV_VIOL_EXPECTED_PARALLEL_CLOSE: return "expected </Parallel> after </Conclusion>";
    default: return "merge without an open block";
  }
}

struct Item {
  int32_t token;
  int32_t source;  // flat index in the forced source stream, -1 otherwise
};

// compile_script (engine.cpp:83-261) over token ids: the lane split of a forced stream.  The label
// text check of :203-210 needs the tokenizer's text and stays with the caller.
struct ScriptLane {
  int parent = -1, ordinal = 0;
  int path_open_source = -1, label_source = -1;
  std::vector<Item> items;
  struct Spawn {
    size_t after_item = 0;
    std::vector<int> children;
    int conclusion_source = -1;
  };
  std::vector<Spawn> spawns;
};

bool compile_script(const int32_t* src, int n, std::vector<ScriptLane>& lanes, std::string& err) {
  enum Phase { AwaitGoal, Goal, AwaitPath, InPath, Conclusion, AwaitClose };
  struct Ctx {
    Phase phase = AwaitGoal;
    int parent = 0, outlines = 0, paths_seen = 0, child = -1;
    bool in_outline = false, after_outline = false, awaiting_label = false;
    size_t spawn_index = 0;
  };
  lanes.assign(1, ScriptLane{});
  std::vector<Ctx> stack;
  auto is_tag = [](int t) { return t >= 0 && t < kTagCount_; };
  auto name = [&](int t) { return is_tag(t) ? std::string(kTagText[t]) : "w" + std::to_string(t); };
  for (int idx = 0; idx < n; ++idx) {
    const int t = src[idx];
    auto violation = [&](const std::string& msg) {
      err = "token " + std::to_string(idx) + ": " + msg;
      return false;
    };
    auto append = [&](int lane) { lanes[lane].items.push_back({t, idx}); };
    if (stack.empty()) {
      if (!is_tag(t)) {
        append(0);
      } else if (t == kParOpen) {
        append(0);
        stack.push_back(Ctx{});
      } else {
        return violation("unexpected " + name(t) + " outside any block");
      }
      continue;
    }
    Ctx& c = stack.back();
    switch (c.phase) {
      case AwaitGoal:
        if (t != kGoalOpen) return violation("expected <Goal> after <Parallel>");
        append(c.parent);
        c.phase = Goal;
        break;
      case Goal:
        if (!is_tag(t)) {
          if (c.after_outline && !c.in_outline) return violation("text between outlines");
          append(c.parent);
        } else if (t == kOutOpen) {
          if (c.in_outline) return violation("nested <Outline>");
          c.in_outline = true;
          ++c.outlines;
          append(c.parent);
        } else if (t == kOutClose) {
          if (!c.in_outline) return violation("</Outline> without <Outline>");
          c.in_outline = false;
          c.after_outline = true;
          append(c.parent);
        } else if (t == kGoalClose) {
          if (c.in_outline) return violation("</Goal> inside <Outline>");
          if (c.outlines == 0) return violation("</Goal> with zero outlines");
          append(c.parent);
          ScriptLane::Spawn sp;
          sp.after_item = lanes[c.parent].items.size();
          for (int k = 1; k <= c.outlines; ++k) {
            ScriptLane l;
            l.parent = c.parent;
            l.ordinal = k;
            sp.children.push_back((int)lanes.size());
            lanes.push_back(std::move(l));
          }
          Ctx& cc = stack.back();  // lanes grew; the context reference is stable (stack unchanged)
          cc.spawn_index = lanes[cc.parent].spawns.size();
          lanes[cc.parent].spawns.push_back(std::move(sp));
          cc.phase = AwaitPath;
        } else {
          return violation("unexpected " + name(t) + " inside <Goal>");
        }
        break;
      case AwaitPath:
        if (t == kPathOpen) {
          if (c.paths_seen == c.outlines) return violation("more <Path> blocks than outlines");
          const int child = lanes[c.parent].spawns[c.spawn_index].children[c.paths_seen];
          lanes[child].path_open_source = idx;
          c.child = child;
          c.awaiting_label = true;
          c.phase = InPath;
        } else if (t == kConcOpen) {
          if (c.paths_seen < c.outlines)
            return violation("only " + std::to_string(c.paths_seen) + " paths for " + std::to_string(c.outlines) +
                             " outlines");
          lanes[c.parent].spawns[c.spawn_index].conclusion_source = idx;
          c.phase = Conclusion;
        } else if (!is_tag(t)) {
          return violation("stray text between paths");
        } else {
          return violation("unexpected " + name(t) + " between paths");
        }
        break;
      case InPath:
        if (c.awaiting_label) {
          if (is_tag(t)) return violation("path body must begin with its index label");
          lanes[c.child].label_source = idx;
          c.awaiting_label = false;
        } else if (!is_tag(t)) {
          append(c.child);
        } else if (t == kParOpen) {
          append(c.child);
          Ctx nested;
          nested.parent = c.child;
          stack.push_back(nested);
        } else if (t == kPathClose) {
          append(c.child);
          ++c.paths_seen;
          c.child = -1;
          c.phase = AwaitPath;
        } else {
          return violation("unexpected " + name(t) + " inside <Path>");
        }
        break;
      case Conclusion:
        if (!is_tag(t)) {
          append(c.parent);
        } else if (t == kConcClose) {
          append(c.parent);
          c.phase = AwaitClose;
        } else {
          return violation("unexpected " + name(t) + " inside <Conclusion>");
        }
        break;
      case AwaitClose:
        if (t != kParClose) return violation("expected </Parallel> after </Conclusion>");
        append(c.parent);
        stack.pop_back();
        break;
    }
  }
  if (!stack.empty()) {
    err = "token " + std::to_string(n) + ": unterminated block at end of stream";
    return false;
  }
  return true;
}

std::string label_to_prefix(const std::string& label) {  // engine.cpp:73-79
  std::string p = label;
  if (!p.empty() && p.back() == ':') p.pop_back();
  return p + '.';
}

struct Lane {
  enum State { Active, Waiting, Zombie, Done };
  int id = 0, req = 0, parent = -1, ordinal = 0;  // id: index in the engine's flat lane list (= K5 slot)
  State state = Active;
  uint64_t handle = 0;
  int next_position = 0;
  int64_t emitted = 0;
  std::deque<Item> inject;
  const ScriptLane* script = nullptr;
  size_t next_item = 0, next_spawn = 0;
  std::vector<std::vector<int>> spawn_children;
  std::vector<int> spawn_conclusion;
  size_t waiting_on = 0;
  std::string label;
  int last_token = -1;  // greedy argmax of the last logits (free running)
  bool has_logits = false;
  bool injected_now = false;
  Item now{};
};

// RequestRuntime (engine.cpp:417-428): one trajectory, its lanes (flat indices), its script.
struct Request {
  int base = 0;                    // flat index of its root lane (forced: lanes base .. base + script size)
  const int32_t* src = nullptr;    // forced source stream
  int n_src = 0;
  int64_t logit_row0 = 0;          // first row of its logits in the caller's buffer
  std::vector<ScriptLane> script;  // forced mode (stable: built before any lane points into it)
  bool failed = false, done = false;
  int failure = 0;
  std::string detail;
  int64_t emitted = 0;
};

class Engine {
 public:
  Engine(mv_toy* toy, mv_kv_store* store, const mv_engine_options& opt) : toy_(toy), s_(store), opt_(opt) {}
  ~Engine() {
    cudaFree(d_state_);
    cudaFree(d_ones_);
    cudaFree(d_events_);
    cudaFree(d_action_);
    cudaFree(d_arg_);
    cudaFree(d_io_);
    cudaFree(d_logits_);
    cudaFree(d_ids_);
    cudaFreeHost(h_io_);
    cudaFreeHost(h_back_);
    cudaFreeHost(h_logits_);
  }

  // Simulator::run (engine.cpp:481-485) over a batch of requests (run_batch, :952-966, with the toy
  // model attached): forced requests when `offsets` is given, one free-running request otherwise.
  mv_status run(const int32_t* src, const int64_t* offsets, int n_req, bool free_running, const int32_t* prompt,
                int n_prompt, int32_t max_steps, mv_engine_label_fn label_fn, void* label_ctx, float* h_logits,
                mv_engine_event* events, int64_t events_cap, mv_engine_report* rep) {
    std::memset(rep, 0, sizeof *rep);
    free_ = free_running;
    label_fn_ = label_fn;
    label_ctx_ = label_ctx;
    h_logits_out_ = h_logits;
    events_ = events;
    events_cap_ = events_cap;
    rep_ = rep;
    vocab_ = toy_cfg_vocab();
    PagedStore& st = *s_->impl;
    stream_ = st.stream();
    reqs_.resize(free_ ? 1 : n_req);
    for (int r = 0; r < (int)reqs_.size(); ++r) {
      Request& q = reqs_[r];
      q.base = (int)lanes_.size();
      if (!free_) {
        q.src = src + offsets[r];
        q.n_src = (int)(offsets[r + 1] - offsets[r]);
        q.logit_row0 = offsets[r];
        std::string err;
        if (!compile_script(q.src, q.n_src, q.script, err)) {  // run_forced returns a failed report
          fail(r, MV_ENGINE_FAIL_GRAMMAR, err);
          lanes_.emplace_back();  // an inert root keeps the flat indexing simple
          lanes_.back().id = q.base;
          lanes_.back().req = r;
          lanes_.back().state = Lane::Done;
          continue;
        }
        for (size_t i = 0; i < q.script.size(); ++i) {
          Lane l;
          l.id = q.base + (int)i;
          l.req = r;
          l.parent = q.script[i].parent >= 0 ? q.base + q.script[i].parent : -1;
          l.ordinal = q.script[i].ordinal;
          l.script = &q.script[i];
          l.state = i == 0 ? Lane::Active : Lane::Done;
          lanes_.push_back(std::move(l));
        }
      } else {
        if (n_prompt <= 0) {
          fail(r, MV_ENGINE_FAIL_GRAMMAR, "free-running decode needs a non-empty prompt");
          break;
        }
        Lane l;
        l.id = q.base;
        l.req = r;
        for (int i = 0; i < n_prompt; ++i) l.inject.push_back({prompt[i], -1});
        lanes_.push_back(std::move(l));
      }
    }
    if (mv_status e = ensure_lanes(std::max<size_t>(lanes_.size(), 1))) return e;
    for (Request& q : reqs_) {
      if (q.failed) continue;
      if (mv_status e = st.create(&lanes_[q.base].handle)) return e;
      if (mv_status e = mv_interp_init(d_state_ + (size_t)q.base * MV_INTERP_STATE_WORDS, 1, nullptr, stream_))
        return e;
    }
    int64_t steps = 0;
    while (true) {
      bool progressed = false;
      if (mv_status e = step_once(&progressed)) return e;
      if (!progressed) break;
      if (max_steps > 0 && ++steps >= max_steps) {
        for (int r = 0; r < (int)reqs_.size(); ++r)
          if (!reqs_[r].failed && !reqs_[r].done) fail(r, MV_ENGINE_FAIL_LIMIT, "max_steps reached");
        break;
      }
    }
    // finalize (engine.cpp:835-880): the first failed request's kind and detail
    for (const Request& q : reqs_)
      if (q.failed && rep_->status == 0) {
        rep_->status = 1;
        rep_->failure = q.failure;
        std::strncpy(rep_->failure_detail, q.detail.c_str(), sizeof rep_->failure_detail - 1);
      }
    rep_->steps = step_;
    rep_->merges = merges_;
    rep_->spawns = spawns_;
    rep_->total_tokens = total_tokens_;
    rep_->lanes = (int64_t)lanes_.size();
    rep_->events = n_events_;
    for (auto& l : lanes_)
      if (l.handle) st.release(l.handle);
    return MV_OK;
  }

 private:
  int toy_cfg_vocab();

  // fail (engine.cpp:804-815): the request stops; other requests go on
  void fail(int r, int kind, const std::string& detail) {
    Request& q = reqs_[r];
    q.failed = true;
    q.failure = kind;
    q.detail = detail;
    for (auto& l : lanes_)
      if (l.req == r && (l.state == Lane::Active || l.state == Lane::Waiting)) l.state = Lane::Done;
    log(MV_EVT_FAILED, r, q.base, -1, -1);
  }

  void log(int kind, int req, int lane, int token, int source) {
    if (events_ && n_events_ < events_cap_) events_[n_events_] = {step_, req, lane - reqs_[req].base, kind, token, source};
    ++n_events_;
  }

  mv_status ensure_lanes(size_t need) {
    if (need <= cap_lanes_) return MV_OK;
    size_t cap = std::max<size_t>(need * 2, 64);
    int32_t* ns = nullptr;
    MV_CUDA_TRY(cudaMalloc(&ns, sizeof(int32_t) * MV_INTERP_STATE_WORDS * cap));
    if (d_state_) {
      MV_CUDA_TRY(cudaMemcpyAsync(ns, d_state_, sizeof(int32_t) * MV_INTERP_STATE_WORDS * cap_lanes_,
                                  cudaMemcpyDeviceToDevice, stream_));
      MV_CUDA_TRY(cudaStreamSynchronize(stream_));
      cudaFree(d_state_);
    }
    d_state_ = ns;
    cudaFree(d_ones_);
    cudaFree(d_events_);
    cudaFree(d_action_);
    cudaFree(d_arg_);
    cudaFree(d_io_);
    cudaFree(d_logits_);
    cudaFree(d_ids_);
    // host staging keeps its contents: a spawn grows the lane set while the step's read-back
    // (actions, ids, logits) is still being consumed
    std::vector<int32_t> back_keep(h_back_ ? h_back_ : (int32_t*)nullptr,
                                   h_back_ ? h_back_ + 3 * cap_lanes_ : (int32_t*)nullptr);
    std::vector<float> logits_keep(h_logits_ ? h_logits_ : (float*)nullptr,
                                   h_logits_ ? h_logits_ + cap_lanes_ * vocab_ : (float*)nullptr);
    const size_t old_cap = cap_lanes_;
    cudaFreeHost(h_io_);
    cudaFreeHost(h_back_);
    cudaFreeHost(h_logits_);
    h_logits_ = nullptr;
    MV_CUDA_TRY(cudaMalloc(&d_ones_, sizeof(int32_t) * cap));
    std::vector<int32_t> ones(cap, 1);
    MV_CUDA_TRY(cudaMemcpy(d_ones_, ones.data(), sizeof(int32_t) * cap, cudaMemcpyHostToDevice));
    MV_CUDA_TRY(cudaMalloc(&d_events_, sizeof(int32_t) * cap));
    MV_CUDA_TRY(cudaMalloc(&d_action_, sizeof(int32_t) * cap));
    MV_CUDA_TRY(cudaMalloc(&d_arg_, sizeof(int32_t) * cap));
    MV_CUDA_TRY(cudaMalloc(&d_io_, sizeof(int32_t) * 2 * cap));
    MV_CUDA_TRY(cudaMalloc(&d_logits_, sizeof(float) * cap * vocab_));
    MV_CUDA_TRY(cudaMalloc(&d_ids_, sizeof(int32_t) * cap));
    MV_CUDA_TRY(cudaMallocHost(&h_io_, sizeof(int32_t) * 3 * cap));
    MV_CUDA_TRY(cudaMallocHost(&h_back_, sizeof(int32_t) * 3 * cap));
    if (h_logits_out_) MV_CUDA_TRY(cudaMallocHost(&h_logits_, sizeof(float) * cap * vocab_));
    // old layout [action | arg | ids] at stride old_cap -> the same rows at stride cap
    for (int r = 0; r < 3 && old_cap; ++r)
      std::memcpy(h_back_ + r * cap, back_keep.data() + r * old_cap, sizeof(int32_t) * old_cap);
    if (h_logits_ && !logits_keep.empty()) std::memcpy(h_logits_, logits_keep.data(), sizeof(float) * logits_keep.size());
    cap_lanes_ = cap;
    return MV_OK;
  }

  // Simulator::step_once (engine.cpp:498-525) with step_lane (:528-582) and emit (:599-677) batched over
  // every active lane of every request.
  mv_status step_once(bool* progressed) {
    *progressed = false;
    std::vector<int> batch;
    const size_t count = lanes_.size();  // lanes spawned in this step start on the next one
    bool any = false;
    for (size_t li = 0; li < count; ++li) any = any || lanes_[li].state == Lane::Active;
    if (!any) return MV_OK;
    ++step_;
    for (size_t li = 0; li < count; ++li) {
      Lane& l = lanes_[li];
      if (l.state != Lane::Active || reqs_[l.req].failed) continue;
      Item it;
      bool injected = false;
      if (!l.inject.empty()) {
        it = l.inject.front();
        l.inject.pop_front();
        injected = true;
      } else if (l.script && l.next_item < l.script->items.size()) {
        it = l.script->items[l.next_item++];
      } else if (free_) {
        if (!l.has_logits) {
          fail(l.req, MV_ENGINE_FAIL_GRAMMAR, "free-running lane has no context to decode from");
          continue;
        }
        it = {l.last_token, -1};
      } else {
        finish_lane(l);
        continue;
      }
      l.now = it;
      l.injected_now = injected;
      batch.push_back((int)li);
    }
    *progressed = true;
    // a request that failed while the batch was being gathered emits nothing this step
    batch.erase(std::remove_if(batch.begin(), batch.end(), [&](int li) { return reqs_[lanes_[li].req].failed; }),
                batch.end());
    const int b = (int)batch.size();
    if (b > 0) {
      // ---- device: one pass for every emitting lane of every request ----
      std::vector<uint64_t> hs(b);
      for (int k = 0; k < b; ++k) {
        Lane& l = lanes_[batch[k]];
        hs[k] = l.handle;
        h_io_[k] = l.now.token;
        h_io_[b + k] = l.next_position;
      }
      const size_t nl = lanes_.size();
      for (size_t li = 0; li < nl; ++li) h_io_[2 * b + li] = MV_INTERP_IDLE;
      for (int k = 0; k < b; ++k) h_io_[2 * b + batch[k]] = lanes_[batch[k]].now.token;
      MV_CUDA_TRY(cudaMemcpyAsync(d_io_, h_io_, sizeof(int32_t) * 2 * b, cudaMemcpyHostToDevice, stream_));
      MV_CUDA_TRY(cudaMemcpyAsync(d_events_, h_io_ + 2 * b, sizeof(int32_t) * nl, cudaMemcpyHostToDevice, stream_));
      if (mv_status e = mv_toy_step(toy_, s_, hs.data(), b, d_io_, d_io_ + b, d_logits_, nullptr, nullptr)) return e;
      if (mv_status e = mv_argmax_rows(d_logits_, b, vocab_, d_ids_, stream_)) return e;
      if (mv_status e = mv_interp_feed(d_state_, (int32_t)nl, d_events_, 1, d_action_, d_arg_, nullptr, nullptr,
                                       stream_))
        return e;
      MV_CUDA_TRY(cudaMemcpyAsync(h_back_, d_action_, sizeof(int32_t) * nl, cudaMemcpyDeviceToHost, stream_));
      MV_CUDA_TRY(cudaMemcpyAsync(h_back_ + cap_lanes_, d_arg_, sizeof(int32_t) * nl, cudaMemcpyDeviceToHost, stream_));
      MV_CUDA_TRY(cudaMemcpyAsync(h_back_ + 2 * cap_lanes_, d_ids_, sizeof(int32_t) * b, cudaMemcpyDeviceToHost,
                                  stream_));
      if (h_logits_out_)
        MV_CUDA_TRY(cudaMemcpyAsync(h_logits_, d_logits_, sizeof(float) * b * vocab_, cudaMemcpyDeviceToHost, stream_));
      MV_CUDA_TRY(cudaStreamSynchronize(stream_));
      // ---- host: emit bookkeeping and interpreter actions, lane order (engine.cpp:643-677) ----
      for (int k = 0; k < b; ++k) {
        Lane& l = lanes_[batch[k]];
        Request& q = reqs_[l.req];
        if (q.failed) continue;  // an earlier lane of this request failed in this step
        if (h_logits_out_ && l.now.source >= 0)
          std::memcpy(h_logits_out_ + (size_t)(q.logit_row0 + l.now.source) * vocab_, h_logits_ + (size_t)k * vocab_,
                      sizeof(float) * vocab_);
        l.last_token = h_back_[2 * cap_lanes_ + k];
        l.has_logits = true;
        ++l.next_position;
        ++l.emitted;
        ++total_tokens_;
        ++q.emitted;
        log(l.injected_now ? MV_EVT_PREFILL : MV_EVT_DECODE, l.req, l.id, l.now.token, l.now.source);
        if (q.emitted > (int64_t)max_request_tokens()) {
          fail(l.req, MV_ENGINE_FAIL_LIMIT, "request exceeded " + std::to_string(max_request_tokens()) + " tokens");
          continue;
        }
        const int act = h_back_[l.id], arg = h_back_[cap_lanes_ + l.id];
        if (act == MV_ACT_VIOLATION) {
          fail(l.req, MV_ENGINE_FAIL_GRAMMAR, violation_text(arg, l.now.token));
          continue;
        }
        if (act == MV_ACT_WORKER_DONE) {
          enter_zombie(l);
          continue;
        }
        if (act == MV_ACT_SPAWN) {
          if (mv_status e = spawn_children(batch[k], arg)) return e;
          continue;
        }
        if (l.parent >= 0 && l.state == Lane::Active && l.emitted >= (int64_t)max_worker_tokens()) enter_zombie(l);
        // script exhausted right after its last token: retire now (engine.cpp:573-579)
        if (l.state == Lane::Active && l.inject.empty() && l.script && l.next_item >= l.script->items.size() &&
            l.next_spawn >= l.script->spawns.size() && !free_)
          finish_lane(l);
      }
    }
    // ---- end of step: merge every waiting lane whose children are all zombies (engine.cpp:516-523) ----
    for (size_t li = 0; li < lanes_.size(); ++li)
      if (lanes_[li].state == Lane::Waiting && !reqs_[lanes_[li].req].failed)
        if (mv_status e = maybe_merge((int)li)) return e;
    return MV_OK;
  }

  size_t max_worker_tokens() const { return opt_.max_worker_tokens > 0 ? (size_t)opt_.max_worker_tokens : 4096; }
  size_t max_request_tokens() const { return opt_.max_request_tokens > 0 ? (size_t)opt_.max_request_tokens : 4096; }

  // spawn_children (engine.cpp:679-725): fork the lane's KV into `count` children that start at its
  // next position with an injected <Path> and their index label.  (lanes_ may grow: indices only.)
  mv_status spawn_children(int pid, int count) {
    const ScriptLane::Spawn* sp = nullptr;
    {
      Lane& l = lanes_[pid];
      if (l.script && l.next_spawn < l.script->spawns.size()) sp = &l.script->spawns[l.next_spawn++];
    }
    std::vector<uint64_t> forks(count);
    if (mv_status e = s_->impl->fork(lanes_[pid].handle, count, forks.data())) return e;
    const int r = lanes_[pid].req, base = reqs_[r].base;
    const std::string prefix = lanes_[pid].label.empty() ? "" : label_to_prefix(lanes_[pid].label);
    std::vector<int> kids;
    for (int k = 1; k <= count; ++k) {
      int cid;
      if (sp) {
        cid = base + sp->children[k - 1];
      } else {
        cid = (int)lanes_.size();
        lanes_.emplace_back();
        lanes_.back().id = cid;
        lanes_.back().req = r;
      }
      kids.push_back(cid);
    }
    if (mv_status e = ensure_lanes(lanes_.size())) return e;
    Lane& p = lanes_[pid];
    for (int k = 1; k <= count; ++k) {
      Lane& c = lanes_[kids[k - 1]];
      c.parent = p.id;
      c.ordinal = k;
      c.state = Lane::Active;
      c.handle = forks[k - 1];
      c.next_position = p.next_position;  // siblings share the start position
      if (c.label.empty()) c.label = prefix + std::to_string(k) + ":";
      const ScriptLane* cl = c.script;
      int label_tok;
      if (cl && cl->label_source >= 0) label_tok = reqs_[r].src[cl->label_source];
      else if (label_fn_) label_tok = label_fn_(label_ctx_, c.label.c_str());
      else label_tok = -1;
      c.inject.push_back({kPathOpen, cl ? cl->path_open_source : -1});
      c.inject.push_back({label_tok, cl ? cl->label_source : -1});
      if (mv_status e = mv_interp_init(d_state_ + (size_t)c.id * MV_INTERP_STATE_WORDS, 1, d_ones_, stream_)) return e;
    }
    p.spawn_children.push_back(kids);
    p.spawn_conclusion.push_back(sp ? sp->conclusion_source : -1);
    p.waiting_on = p.spawn_children.size() - 1;
    p.state = Lane::Waiting;
    ++spawns_;
    log(MV_EVT_SPAWN, r, p.id, count, -1);
    return MV_OK;
  }

  void enter_zombie(Lane& l) {
    l.state = Lane::Zombie;
    log(MV_EVT_ZOMBIE, l.req, l.id, -1, -1);
  }

  void finish_lane(Lane& l);

  // maybe_merge (engine.cpp:767-802)
  mv_status maybe_merge(int li) {
    Lane& l = lanes_[li];
    const std::vector<int>& kids = l.spawn_children[l.waiting_on];
    std::vector<uint64_t> branches;
    for (int c : kids) {
      if (lanes_[c].state != Lane::Zombie) return MV_OK;
      branches.push_back(lanes_[c].handle);
    }
    uint64_t merged = 0;
    if (mv_status e = s_->impl->merge(l.handle, branches.data(), (int32_t)branches.size(), &merged)) return e;
    ++merges_;
    if (mv_status e = s_->impl->release(l.handle)) return e;
    for (int c : kids) {
      Lane& ch = lanes_[c];
      if (mv_status e = s_->impl->release(ch.handle)) return e;
      ch.handle = 0;
      ch.state = Lane::Done;
      l.next_position = std::max(l.next_position, ch.next_position);
    }
    l.handle = merged;
    // the interpreter's frame resumes at AwaitConclusionTag (engine.cpp:793): a MERGED event
    std::vector<int32_t> ev(lanes_.size(), MV_INTERP_IDLE);
    ev[l.id] = MV_INTERP_MERGED;
    MV_CUDA_TRY(cudaMemcpyAsync(d_events_, ev.data(), sizeof(int32_t) * ev.size(), cudaMemcpyHostToDevice, stream_));
    if (mv_status e = mv_interp_feed(d_state_, (int32_t)ev.size(), d_events_, 1, d_action_, d_arg_, nullptr, nullptr,
                                     stream_))
      return e;
    MV_CUDA_TRY(cudaStreamSynchronize(stream_));  // ev is pageable host memory
    l.inject.push_back({kConcOpen, l.spawn_conclusion[l.waiting_on]});
    l.state = Lane::Active;
    log(MV_EVT_MERGE, l.req, l.id, -1, -1);
    return MV_OK;
  }

  mv_toy* toy_;
  mv_kv_store* s_;
  mv_engine_options opt_;
  cudaStream_t stream_ = nullptr;
  bool free_ = false;
  mv_engine_label_fn label_fn_ = nullptr;
  void* label_ctx_ = nullptr;
  float* h_logits_out_ = nullptr;
  mv_engine_event* events_ = nullptr;
  int64_t events_cap_ = 0, n_events_ = 0;
  mv_engine_report* rep_ = nullptr;
  int vocab_ = 0;
  std::deque<Request> reqs_;  // stable addresses: lanes point into their request's script
  std::vector<Lane> lanes_;
  int64_t step_ = 0, merges_ = 0, spawns_ = 0, total_tokens_ = 0;
  size_t cap_lanes_ = 0;
  int32_t *d_state_ = nullptr, *d_ones_ = nullptr, *d_events_ = nullptr, *d_action_ = nullptr, *d_arg_ = nullptr;
  int32_t *d_io_ = nullptr, *d_ids_ = nullptr;
  float* d_logits_ = nullptr;
  int32_t *h_io_ = nullptr, *h_back_ = nullptr;
  float* h_logits_ = nullptr;
};

// finish_lane (engine.cpp:750-765): a root lane whose stream ended with a block still open fails
void Engine::finish_lane(Lane& l) {
  if (l.parent < 0) {
    l.state = Lane::Done;
    int32_t st[MV_INTERP_STATE_WORDS] = {0, 0};
    cudaMemcpyAsync(st, d_state_ + (size_t)l.id * MV_INTERP_STATE_WORDS, sizeof st, cudaMemcpyDeviceToHost, stream_);
    cudaStreamSynchronize(stream_);
    if ((st[0] & 0xff) == 0) {
      reqs_[l.req].done = true;
      log(MV_EVT_DONE, l.req, l.id, -1, -1);
    } else {
      fail(l.req, MV_ENGINE_FAIL_GRAMMAR, "stream ended inside an open block");
    }
  } else {
    fail(l.req, MV_ENGINE_FAIL_GRAMMAR, "worker stream ended early");
  }
}

}  // namespace
}  // namespace mv

using namespace mv;

int Engine::toy_cfg_vocab() { return mv_toy_vocab(toy_); }

static mv_status engine_store(mv_toy* toy, const mv_engine_options* opt, mv_kv_store** out) {
  mv_toy_config c{};
  if (mv_status e = mv_toy_get_config(toy, &c)) return e;
  mv_kv_config kc{};
  kc.num_pages = opt && opt->num_pages > 0 ? opt->num_pages : 4096;
  kc.layers = c.layers;
  kc.kv_heads = c.heads;
  kc.head_dim = mv_attn_head_dim(c.model_dim / c.heads);
  kc.rope_base = c.rope_base;
  return mv_kv_store_create(&kc, out);
}

extern "C" mv_status mv_engine_run_batch(mv_toy* toy, const int32_t* h_tokens, const int64_t* h_offsets, int32_t n_req,
                                         const mv_engine_options* opt, mv_stream_t stream, float* h_logits,
                                         mv_engine_event* h_events, int64_t events_cap, mv_engine_report* rep) {
  if (!toy || !rep || n_req < 1 || !h_offsets || (h_offsets[n_req] > 0 && !h_tokens))
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_engine_run_batch: bad arguments");
  for (int r = 0; r < n_req; ++r)
    if (h_offsets[r + 1] < h_offsets[r]) return fail(MV_ERR_INVALID_ARGUMENT, "mv_engine_run_batch: bad offsets");
  mv_engine_options o{};
  if (opt) o = *opt;
  mv_kv_store* s = nullptr;
  if (mv_status e = engine_store(toy, &o, &s)) return e;
  mv_kv_set_stream(s, stream);
  mv_status st;
  {
    Engine eng(toy, s, o);
    st = eng.run(h_tokens, h_offsets, n_req, false, nullptr, 0, 0, nullptr, nullptr, h_logits, h_events, events_cap,
                 rep);
  }
  mv_kv_store_destroy(s);
  return st;
}

extern "C" mv_status mv_engine_run_forced(mv_toy* toy, const int32_t* h_tokens, int32_t n,
                                          const mv_engine_options* opt, mv_stream_t stream, float* h_logits,
                                          mv_engine_event* h_events, int64_t events_cap, mv_engine_report* rep) {
  if (n < 0) return fail(MV_ERR_INVALID_ARGUMENT, "mv_engine_run_forced: n < 0");
  const int64_t offs[2] = {0, n};
  return mv_engine_run_batch(toy, h_tokens, offs, 1, opt, stream, h_logits, h_events, events_cap, rep);
}

extern "C" mv_status mv_engine_run_free(mv_toy* toy, const int32_t* h_prompt, int32_t n_prompt, int32_t max_steps,
                                        const mv_engine_options* opt, mv_engine_label_fn label_fn, void* label_ctx,
                                        mv_stream_t stream, mv_engine_event* h_events, int64_t events_cap,
                                        mv_engine_report* rep) {
  if (!toy || !rep || n_prompt < 0 || (n_prompt > 0 && !h_prompt))
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_engine_run_free: bad arguments");
  mv_engine_options o{};
  if (opt) o = *opt;
  mv_kv_store* s = nullptr;
  if (mv_status e = engine_store(toy, &o, &s)) return e;
  mv_kv_set_stream(s, stream);
  mv_status st;
  {
    Engine eng(toy, s, o);
    st = eng.run(nullptr, nullptr, 1, true, h_prompt, n_prompt, max_steps, label_fn, label_ctx, nullptr, h_events,
                 events_cap, rep);
  }
  mv_kv_store_destroy(s);
  return st;
}
