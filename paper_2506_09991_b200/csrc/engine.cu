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
  int id = 0, parent = -1, ordinal = 0;
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

  mv_status run(const int32_t* src, int n, bool free_running, const int32_t* prompt, int n_prompt, int32_t max_steps,
                mv_engine_label_fn label_fn, void* label_ctx, float* h_logits, mv_engine_event* events,
                int64_t events_cap, mv_engine_report* rep) {
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
    if (!free_) {
      std::string err;
      if (!compile_script(src, n, script_, err)) return failed(MV_ENGINE_FAIL_GRAMMAR, err), MV_OK;
      lanes_.resize(script_.size());
      for (size_t i = 0; i < script_.size(); ++i) {
        lanes_[i].id = (int)i;
        lanes_[i].parent = script_[i].parent;
        lanes_[i].ordinal = script_[i].ordinal;
        lanes_[i].script = &script_[i];
        lanes_[i].state = i == 0 ? Lane::Active : Lane::Done;
      }
    } else {
      if (n_prompt <= 0) return failed(MV_ENGINE_FAIL_GRAMMAR, "free-running decode needs a non-empty prompt"), MV_OK;
      lanes_.resize(1);
      for (int i = 0; i < n_prompt; ++i) lanes_[0].inject.push_back({prompt[i], -1});
    }
    if (mv_status e = st.create(&lanes_[0].handle)) return e;
    if (mv_status e = ensure_lanes(lanes_.size())) return e;
    if (mv_status e = mv_interp_init(d_state_, 1, nullptr, stream_)) return e;
    int64_t steps = 0;
    while (true) {
      bool progressed = false;
      if (mv_status e = step_once(&progressed)) return e;
      if (!progressed) break;
      if (max_steps > 0 && ++steps >= max_steps) break;
    }
    if (!failed_ && !done_) {  // the loop stopped with no active lane (or at max_steps)
      bool active = false;
      for (auto& l : lanes_) active = active || l.state == Lane::Active || l.state == Lane::Waiting;
      if (active && max_steps > 0) failed(MV_ENGINE_FAIL_LIMIT, "max_steps reached");
    }
    rep_->status = failed_ ? 1 : 0;
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

  void failed(int kind, const std::string& detail) {
    failed_ = true;
    rep_->failure = kind;
    std::strncpy(rep_->failure_detail, detail.c_str(), sizeof rep_->failure_detail - 1);
    for (auto& l : lanes_)
      if (l.state == Lane::Active || l.state == Lane::Waiting) l.state = Lane::Done;
    log(MV_EVT_FAILED, 0, -1, -1);
  }

  void log(int kind, int lane, int token, int source) {
    if (events_ && n_events_ < events_cap_) events_[n_events_] = {step_, lane, kind, token, source};
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

  // Simulator::step_once (engine.cpp:498-525) with step_lane (:528-582) and emit (:599-677) batched.
  mv_status step_once(bool* progressed) {
    *progressed = false;
    if (failed_ || done_) return MV_OK;
    std::vector<int> batch;
    const size_t count = lanes_.size();  // lanes spawned in this step start on the next one
    bool any = false;
    for (size_t li = 0; li < count; ++li) any = any || lanes_[li].state == Lane::Active;
    if (!any) return MV_OK;
    ++step_;
    for (size_t li = 0; li < count && !failed_; ++li) {
      Lane& l = lanes_[li];
      if (l.state != Lane::Active) continue;
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
          failed(MV_ENGINE_FAIL_GRAMMAR, "free-running lane has no context to decode from");
          break;
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
    if (failed_) return MV_OK;
    *progressed = true;
    const int b = (int)batch.size();
    if (b > 0) {
      // ---- device: one pass for every emitting lane ----
      std::vector<uint64_t> hs(b);
      for (int k = 0; k < b; ++k) {
        Lane& l = lanes_[batch[k]];
        hs[k] = l.handle;
        h_io_[k] = l.now.token;
        h_io_[b + k] = l.next_position;
      }
      for (size_t li = 0; li < lanes_.size(); ++li) h_io_[2 * b + li] = MV_INTERP_IDLE;
      for (int k = 0; k < b; ++k) h_io_[2 * b + batch[k]] = lanes_[batch[k]].now.token;
      const size_t nl = lanes_.size();
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
      for (int k = 0; k < b && !failed_; ++k) {
        Lane& l = lanes_[batch[k]];
        if (h_logits_out_ && l.now.source >= 0)
          std::memcpy(h_logits_out_ + (size_t)l.now.source * vocab_, h_logits_ + (size_t)k * vocab_,
                      sizeof(float) * vocab_);
        l.last_token = h_back_[2 * cap_lanes_ + k];
        l.has_logits = true;
        ++l.next_position;
        ++l.emitted;
        ++total_tokens_;
        ++req_emitted_;
        log(l.injected_now ? MV_EVT_PREFILL : MV_EVT_DECODE, l.id, l.now.token, l.now.source);
        if (req_emitted_ > (int64_t)max_request_tokens()) {
          failed(MV_ENGINE_FAIL_LIMIT, "request exceeded " + std::to_string(max_request_tokens()) + " tokens");
          break;
        }
        const int act = h_back_[l.id], arg = h_back_[cap_lanes_ + l.id];
        if (act == MV_ACT_VIOLATION) {
          failed(MV_ENGINE_FAIL_GRAMMAR, violation_text(arg, l.now.token));
          break;
        }
        if (act == MV_ACT_WORKER_DONE) {
          enter_zombie(l);
          continue;
        }
        if (act == MV_ACT_SPAWN) {
          if (mv_status e = spawn_children(l, arg)) return e;
          continue;
        }
        if (l.parent >= 0 && l.state == Lane::Active && l.emitted >= (int64_t)max_worker_tokens()) enter_zombie(l);
        // script exhausted right after its last token: retire now (engine.cpp:573-579)
        if (l.state == Lane::Active && l.inject.empty() && l.script && l.next_item >= l.script->items.size() &&
            l.next_spawn >= l.script->spawns.size() && !free_)
          finish_lane(l);
      }
    }
    if (failed_) return MV_OK;
    // ---- end of step: merge every waiting lane whose children are all zombies (engine.cpp:516-523) ----
    for (size_t li = 0; li < lanes_.size(); ++li)
      if (lanes_[li].state == Lane::Waiting)
        if (mv_status e = maybe_merge(lanes_[li])) return e;
    return MV_OK;
  }

  size_t max_worker_tokens() const { return opt_.max_worker_tokens > 0 ? (size_t)opt_.max_worker_tokens : 4096; }
  size_t max_request_tokens() const { return opt_.max_request_tokens > 0 ? (size_t)opt_.max_request_tokens : 4096; }

  // spawn_children (engine.cpp:679-725): fork the lane's KV into `count` children that start at its
  // next position with an injected <Path> and their index label.
  mv_status spawn_children(Lane& l, int count) {
    const int pid = l.id;  // lanes_ may grow below: the parent is re-fetched by index
    const ScriptLane::Spawn* sp = nullptr;
    if (l.script && l.next_spawn < l.script->spawns.size()) sp = &l.script->spawns[l.next_spawn++];
    std::vector<uint64_t> forks(count);
    if (mv_status e = s_->impl->fork(l.handle, count, forks.data())) return e;
    const std::string prefix = l.label.empty() ? "" : label_to_prefix(l.label);
    std::vector<int> kids;
    for (int k = 1; k <= count; ++k) {
      int cid;
      if (sp) {
        cid = sp->children[k - 1];
      } else {
        cid = (int)lanes_.size();
        lanes_.emplace_back();
        lanes_.back().id = cid;
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
      if (cl && cl->label_source >= 0) label_tok = src_token(cl->label_source);
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
    log(MV_EVT_SPAWN, p.id, count, -1);
    return MV_OK;
  }

  int src_token(int source) const { return source >= 0 && source < n_src_ ? src_[source] : -1; }

  void enter_zombie(Lane& l) {
    l.state = Lane::Zombie;
    log(MV_EVT_ZOMBIE, l.id, -1, -1);
  }

  void finish_lane(Lane& l);

  // maybe_merge (engine.cpp:767-802)
  mv_status maybe_merge(Lane& l) {
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
    log(MV_EVT_MERGE, l.id, -1, -1);
    return MV_OK;
  }

 public:
  const int32_t* src_ = nullptr;
  int n_src_ = 0;

 private:
  mv_toy* toy_;
  mv_kv_store* s_;
  mv_engine_options opt_;
  cudaStream_t stream_ = nullptr;
  bool free_ = false, failed_ = false, done_ = false;
  mv_engine_label_fn label_fn_ = nullptr;
  void* label_ctx_ = nullptr;
  float* h_logits_out_ = nullptr;
  mv_engine_event* events_ = nullptr;
  int64_t events_cap_ = 0, n_events_ = 0;
  mv_engine_report* rep_ = nullptr;
  int vocab_ = 0;
  std::vector<ScriptLane> script_;
  std::vector<Lane> lanes_;
  int64_t step_ = 0, merges_ = 0, spawns_ = 0, total_tokens_ = 0, req_emitted_ = 0;
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
      done_ = true;
      log(MV_EVT_DONE, l.id, -1, -1);
    } else {
      failed(MV_ENGINE_FAIL_GRAMMAR, "stream ended inside an open block");
    }
  } else {
    failed(MV_ENGINE_FAIL_GRAMMAR, "worker stream ended early");
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
  kc.head_dim = kHeadDim;
  kc.rope_base = c.rope_base;
  return mv_kv_store_create(&kc, out);
}

extern "C" mv_status mv_engine_run_forced(mv_toy* toy, const int32_t* h_tokens, int32_t n,
                                          const mv_engine_options* opt, mv_stream_t stream, float* h_logits,
                                          mv_engine_event* h_events, int64_t events_cap, mv_engine_report* rep) {
  if (!toy || !rep || (n > 0 && !h_tokens) || n < 0) return fail(MV_ERR_INVALID_ARGUMENT, "mv_engine_run_forced: bad arguments");
  mv_engine_options o{};
  if (opt) o = *opt;
  mv_kv_store* s = nullptr;
  if (mv_status e = engine_store(toy, &o, &s)) return e;
  mv_kv_set_stream(s, stream);
  mv_status st;
  {
    Engine eng(toy, s, o);
    eng.src_ = h_tokens;
    eng.n_src_ = n;
    st = eng.run(h_tokens, n, false, nullptr, 0, 0, nullptr, nullptr, h_logits, h_events, events_cap, rep);
  }
  mv_kv_store_destroy(s);
  return st;
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
    st = eng.run(nullptr, 0, true, h_prompt, n_prompt, max_steps, label_fn, label_ctx, nullptr, h_events, events_cap,
                 rep);
  }
  mv_kv_store_destroy(s);
  return st;
}
