// TEST INFRASTRUCTURE ONLY (oracle/). Golden-vector generator and CPU-baseline driver
// linked against the *patched reference core* that oracle/ref_build.sh compiles from
// /root/reference/proj/core into oracle/_ref/. Nothing in the product links this file.
//
// Modes (all write JSON lines to stdout):
//   refdrv dag <fixtures_dir>        build_dag/assign_positions/build_mask goldens
//                                    (dag.cpp:198-263) for the shipped fixtures, seeded
//                                    synth::random_trajectory inputs (synth.cpp:94-114) and
//                                    malformed mutations (grammar.cpp:156-294 ParseError kinds)
//   refdrv kv <seed> <ops> <rec>     seeded RadixStore op logs (kvcache.cpp:90-397) with the
//                                    reference's outcome of every op
//   refdrv toy                       ToyModel step/forward and engine::run_forced goldens
//                                    (toy_model.cpp:83-202, engine.cpp:928-939)
//   refdrv forced <words> <plen>     time engine::run_forced on the C1 config (BASELINE
//                                    configs[0]); prints tokens/s
//   refdrv decode <threads> <secs>   time the reference decode path (resolve_payloads + step)
//                                    on the configs[1] shape; prints tokens/s
//   refdrv c5 <rounds> <rec_bytes>   time RadixStore fork / extend / merge / release on the
//                                    configs[4] protocol (prefix 4096; per round fork 128,
//                                    64 tokens per branch, ordinal merge, 16 Reduce tokens)
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "multiverse/dag.hpp"
#include "multiverse/engine.hpp"
#include "multiverse/grammar.hpp"
#include "multiverse/kvcache.hpp"
#include "multiverse/synth.hpp"
#include "multiverse/tokenizer.hpp"
#include "multiverse/toy_model.hpp"

using namespace multiverse;

namespace {

std::string read_file(const std::string& p) {
  std::ifstream in(p, std::ios::binary);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

template <typename T>
void put_vec(const char* key, const std::vector<T>& v) {
  std::printf("\"%s\":[", key);
  for (std::size_t i = 0; i < v.size(); ++i) {
    if (i) std::printf(",");
    if constexpr (std::is_floating_point_v<T>) {
      std::printf("%.17g", static_cast<double>(v[i]));
    } else {
      std::printf("%lld", static_cast<long long>(v[i]));
    }
  }
  std::printf("]");
}

std::uint64_t fnv1a(const std::uint8_t* p, std::size_t n, std::uint64_t h = 1469598103934665603ull) {
  for (std::size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

std::string json_escape(const std::string& s) {
  std::string o;
  for (char c : s) {
    if (c == '"' || c == '\\') {
      o += '\\';
      o += c;
    } else if (c == '\n') {
      o += "\\n";
    } else if (static_cast<unsigned char>(c) < 0x20) {
      char b[8];
      std::snprintf(b, sizeof b, "\\u%04x", c);
      o += b;
    } else {
      o += c;
    }
  }
  return o;
}

// ---------------------------------------------------------------------------
// dag goldens
// ---------------------------------------------------------------------------
void emit_dag_case(const std::string& name, const std::string& text, bool dense) {
  tok::Tokenizer tz;
  std::vector<int> ids;
  for (const auto& t : tz.tokenize(text)) ids.push_back(t.id);
  std::printf("{\"kind\":\"dag\",\"name\":\"%s\",", name.c_str());
  put_vec("tokens", ids);
  try {
    grammar::Trajectory traj = grammar::parse_text(text);
    tok::Tokenizer tz2;
    dag::GenerationDag g = dag::build_dag(traj, tz2);
    dag::VisibilitySpec spec = dag::build_visibility(g);
    auto rows = g.token_layout();
    std::vector<int> layout_ids, seg, segkind;
    for (auto [sid, off] : rows) {
      const auto& s = g.segments[static_cast<std::size_t>(sid)];
      layout_ids.push_back(s.tokens[static_cast<std::size_t>(off)].id);
      seg.push_back(sid);
      segkind.push_back(static_cast<int>(s.kind));
    }
    if (layout_ids != ids) {
      std::fprintf(stderr, "layout ids differ from tokenize() ids for %s\n", name.c_str());
      std::exit(3);
    }
    std::size_t n = rows.size();
    std::vector<std::uint8_t> packed((n * n + 7) / 8, 0);
    for (std::size_t i = 0; i < n; ++i)
      for (std::size_t j = 0; j < n; ++j)
        if (spec.mask.at(i, j)) packed[(i * n + j) >> 3] |= static_cast<std::uint8_t>(0x80u >> ((i * n + j) & 7));
    std::printf(",\"error\":-1,");
    put_vec("positions", spec.positions);
    std::printf(",");
    put_vec("seg", seg);
    std::printf(",");
    put_vec("segkind", segkind);
    std::printf(",\"mask_fnv\":\"%016" PRIx64 "\"", fnv1a(packed.data(), packed.size()));
    if (dense) {
      std::printf(",\"mask_hex\":\"");
      for (auto b : packed) std::printf("%02x", b);
      std::printf("\"");
    }
  } catch (const grammar::ParseError& e) {
    std::printf(",\"error\":%d", static_cast<int>(e.kind()));
  }
  std::printf("}\n");
}

std::string mutate(synth::Rng& rng, const std::string& src, int* which) {
  // Token-level mutations of a well-formed trajectory; each maps to a ParseError
  // (or, rarely, to another well-formed trajectory; the golden records either way).
  static const char* kTags[] = {"<Parallel>", "</Parallel>", "<Goal>", "</Goal>", "<Outline>",
                                "</Outline>", "<Path>", "</Path>", "<Conclusion>", "</Conclusion>"};
  std::vector<std::pair<std::size_t, int>> tags;
  for (std::size_t i = 0; i < src.size(); ++i) {
    if (src[i] != '<') continue;
    for (int k = 0; k < 10; ++k) {
      std::size_t L = std::strlen(kTags[k]);
      if (src.compare(i, L, kTags[k]) == 0) {
        tags.emplace_back(i, k);
        break;
      }
    }
  }
  int m = rng.next_int(0, 3);
  *which = m;
  if (tags.empty()) return src + " </Path>";
  auto [at, k] = tags[static_cast<std::size_t>(rng.next_int(0, static_cast<int>(tags.size()) - 1))];
  std::size_t L = std::strlen(kTags[k]);
  switch (m) {
    case 0:  // drop one tag
      return src.substr(0, at) + src.substr(at + L);
    case 1:  // duplicate one tag
      return src.substr(0, at) + kTags[k] + " " + src.substr(at);
    case 2:  // stray word right after a tag (illegal in whitespace gaps)
      return src.substr(0, at + L) + " stray " + src.substr(at + L);
    default: {  // drop one whole <Path>...</Path> (count mismatch) when possible
      std::size_t p = src.find("<Path>");
      std::size_t q = src.find("</Path>", p == std::string::npos ? 0 : p);
      if (p == std::string::npos || q == std::string::npos) return src.substr(0, at) + src.substr(at + L);
      // only well-formed when the dropped path holds no nested block
      std::string inner = src.substr(p, q - p);
      if (inner.find("<Parallel>") != std::string::npos) return src.substr(0, at) + src.substr(at + L);
      return src.substr(0, p) + src.substr(q + 7);
    }
  }
}

// Every trajectory of the dag goldens: fixtures, seeded random trajectories, malformed mutants.
template <typename F>
void for_each_dag_case(const std::string& fixdir, F&& emit) {
  for (const char* f : {"t1.txt", "nested.txt", "collective_4path.txt", "selective_2path.txt",
                        "generation_collective.txt", "generation_selective.txt", "sequential.txt"}) {
    emit(std::string("fixture:") + f, read_file(fixdir + "/" + f), true);
  }
  for (int seed = 0; seed < 300; ++seed) {
    synth::Rng rng(static_cast<std::uint64_t>(seed));
    synth::TrajectoryParams p;
    p.max_depth = 3;
    p.max_paths = 5;
    emit("random3x5:" + std::to_string(seed), synth::random_trajectory(rng, p), seed < 100);
  }
  for (int seed = 0; seed < 40; ++seed) {
    synth::Rng rng(static_cast<std::uint64_t>(1000 + seed));
    synth::TrajectoryParams p;
    p.max_depth = 4;
    p.max_paths = 6;
    p.max_blocks = 3;
    p.nest_probability = 0.6;
    emit("random4x6:" + std::to_string(seed), synth::random_trajectory(rng, p), false);
  }
  for (int seed = 0; seed < 200; ++seed) {
    synth::Rng rng(static_cast<std::uint64_t>(5000 + seed));
    synth::TrajectoryParams p;
    p.max_depth = 2;
    p.max_paths = 3;
    std::string src = synth::random_trajectory(rng, p);
    int which = 0;
    std::string bad = mutate(rng, src, &which);
    emit("mutant" + std::to_string(which) + ":" + std::to_string(seed), bad, false);
  }
}

int mode_dag(const std::string& fixdir) {
  for_each_dag_case(fixdir, emit_dag_case);
  return 0;
}

// Teacher-forced batch targets (dag.cpp:314-359): target ids and loss masks with and without
// tag loss (BatchOptions::tag_loss), for every parse-valid trajectory of the dag goldens.
void emit_batch_case(const std::string& name, const std::string& text, bool) {
  try {
    grammar::Trajectory traj = grammar::parse_text(text);
    tok::Tokenizer tz;
    dag::GenerationDag g = dag::build_dag(traj, tz);
    dag::BatchOptions with_tags, no_tags;
    no_tags.tag_loss = false;
    dag::TrainingBatch a = dag::build_training_batch(g, with_tags);
    dag::TrainingBatch b = dag::build_training_batch(g, no_tags);
    std::vector<int> la(a.loss_mask.begin(), a.loss_mask.end()), lb(b.loss_mask.begin(), b.loss_mask.end());
    std::printf("{\"kind\":\"batch\",\"name\":\"%s\",", name.c_str());
    put_vec("tokens", a.token_ids);
    std::printf(",");
    put_vec("targets", a.target_ids);
    std::printf(",");
    put_vec("loss_mask", la);
    std::printf(",");
    put_vec("loss_mask_no_tags", lb);
    std::printf("}\n");
  } catch (const grammar::ParseError&) {
  }
}

int mode_batch(const std::string& fixdir) {
  for_each_dag_case(fixdir, emit_batch_case);
  return 0;
}

// ---------------------------------------------------------------------------
// kv op-log goldens
// ---------------------------------------------------------------------------
// Payload of the token at logical index t = FNV-1a over the token prefix [0..t] (8 bytes),
// so a payload is a function of (prefix, token) exactly like real K/V: dedup in the radix
// store and no-dedup in a paged store then resolve to identical bytes.
std::vector<std::byte> payloads_for(const std::vector<kv::TokenId>& base, const std::vector<kv::TokenId>& toks,
                                    std::size_t rec) {
  std::vector<std::byte> out;
  if (rec == 0) return out;
  std::vector<kv::TokenId> seq = base;
  for (auto t : toks) {
    seq.push_back(t);
    std::uint64_t h = fnv1a(reinterpret_cast<const std::uint8_t*>(seq.data()), seq.size() * sizeof(kv::TokenId));
    std::byte b[8];
    std::memcpy(b, &h, 8);
    for (std::size_t k = 0; k < rec; ++k) out.push_back(b[k % 8]);
  }
  return out;
}

int mode_kv(std::uint64_t seed, int n_ops, std::size_t rec) {
  synth::Rng rng(seed);
  kv::RadixStore store(rec);
  std::map<std::uint64_t, std::vector<kv::TokenId>> live;  // flat mirror (tests/oracles.hpp:141-186)
  std::map<std::uint64_t, std::size_t> lens;
  std::vector<std::uint64_t> released;
  // Lineage slots: fresh ids per appended token, copied by fork/merge/extend -- the
  // physical-sharing model of a store that does not dedup. Merges whose reference
  // outcome (slot identity incl. radix dedup) differs from the lineage outcome are
  // skipped, so every logged op has one well-defined answer.
  std::map<std::uint64_t, std::vector<std::uint64_t>> lslots;
  std::uint64_t fresh_slot = 1;
  std::printf("{\"kind\":\"kvlog\",\"seed\":%" PRIu64 ",\"record\":%zu}\n", seed, rec);
  auto pick = [&]() -> std::uint64_t {
    int k = rng.next_int(0, static_cast<int>(live.size()) - 1);
    auto it = live.begin();
    std::advance(it, k);
    return it->first;
  };
  auto emit_resolve = [&](std::uint64_t id) {
    kv::SequenceHandle h{id, lens[id]};
    auto toks = store.resolve(h);
    auto pl = store.resolve_payloads(h);
    std::printf("{\"id\":%" PRIu64 ",", id);
    put_vec("tokens", toks);
    std::printf(",\"payload_fnv\":\"%016" PRIx64 "\"}",
                fnv1a(reinterpret_cast<const std::uint8_t*>(pl.data()), pl.size()));
  };
  for (int op = 0; op < n_ops; ++op) {
    int r = rng.next_int(0, 99);
    std::string kind;
    std::vector<std::uint64_t> args, results;
    std::vector<kv::TokenId> toks;
    int n = 0;
    int err = -1;
    if (live.empty() || r < 6) {
      kind = "create";
      auto h = store.create();
      live[h.id] = {};
      lens[h.id] = 0;
      lslots[h.id] = {};
      results.push_back(h.id);
    } else if (r < 46) {
      kind = "extend";
      std::uint64_t id = pick();
      args.push_back(id);
      int cnt = rng.next_int(0, 20);
      for (int i = 0; i < cnt; ++i) toks.push_back(10 + rng.next_int(0, 5));
      auto pl = payloads_for(live[id], toks, rec);
      if (rec > 0 && !toks.empty()) {
        // Radix dedup may re-trace an edge whose slots hold a payload written under a
        // different context (a merged handle's tail continues inside a branch node); a store
        // without dedup writes the fresh payload instead. Such extends have no single answer
        // across store designs, so they are skipped (dry run on a copy).
        kv::RadixStore probe = store;
        auto ph = probe.extend(kv::SequenceHandle{id, lens[id]}, toks, pl);
        auto got = probe.resolve_payloads(ph);
        if (!std::equal(pl.begin(), pl.end(), got.end() - static_cast<std::ptrdiff_t>(pl.size()))) continue;
      }
      auto h = store.extend(kv::SequenceHandle{id, lens[id]}, toks, pl);
      auto seq = live[id];
      seq.insert(seq.end(), toks.begin(), toks.end());
      live[h.id] = seq;
      lens[h.id] = h.length;
      auto ls = lslots[id];
      for (std::size_t t = 0; t < toks.size(); ++t) ls.push_back(fresh_slot++);
      lslots[h.id] = ls;
      results.push_back(h.id);
    } else if (r < 60) {
      kind = "fork";
      std::uint64_t id = pick();
      args.push_back(id);
      n = rng.next_int(1, 5);
      auto hs = store.fork(kv::SequenceHandle{id, lens[id]}, n);
      for (auto& h : hs) {
        live[h.id] = live[id];
        lens[h.id] = h.length;
        lslots[h.id] = lslots[id];
        results.push_back(h.id);
      }
    } else if (r < 76) {
      kind = "merge";
      std::uint64_t pid = pick();
      args.push_back(pid);
      // branches: descendants by token prefix (engine pattern), occasionally a random one
      std::vector<std::uint64_t> cands;
      for (auto& [id, seq] : live) {
        const auto& ps = live[pid];
        if (seq.size() >= ps.size() && std::equal(ps.begin(), ps.end(), seq.begin())) cands.push_back(id);
      }
      int nb = rng.next_int(1, 4);
      for (int b = 0; b < nb; ++b) {
        if (rng.next_int(0, 9) == 0 || cands.empty()) args.push_back(pick());
        else args.push_back(cands[static_cast<std::size_t>(rng.next_int(0, static_cast<int>(cands.size()) - 1))]);
      }
      std::vector<kv::SequenceHandle> bs;
      for (std::size_t b = 1; b < args.size(); ++b) bs.push_back({args[b], lens[args[b]]});
      {
        bool ref_ok = true, lin_ok = true;
        auto ps = store.resolve_slots(kv::SequenceHandle{pid, lens[pid]});
        const auto& pl = lslots[pid];
        for (std::size_t b = 1; b < args.size(); ++b) {
          if (lens[args[b]] < lens[pid]) { ref_ok = lin_ok = false; break; }
          auto bsl = store.resolve_slots(bs[b - 1]);
          const auto& bl = lslots[args[b]];
          if (!std::equal(ps.begin(), ps.end(), bsl.begin())) ref_ok = false;
          if (!std::equal(pl.begin(), pl.end(), bl.begin())) lin_ok = false;
        }
        if (ref_ok != lin_ok) continue;  // dedup-only sharing: ambiguous across store designs
      }
      try {
        auto h = store.merge(kv::SequenceHandle{pid, lens[pid]}, bs);
        auto seq = live[pid];
        for (std::size_t b = 1; b < args.size(); ++b) {
          const auto& bsq = live[args[b]];
          seq.insert(seq.end(), bsq.begin() + static_cast<std::ptrdiff_t>(live[pid].size()), bsq.end());
        }
        live[h.id] = seq;
        lens[h.id] = h.length;
        auto ls = lslots[pid];
        for (std::size_t b = 1; b < args.size(); ++b) {
          const auto& bl = lslots[args[b]];
          ls.insert(ls.end(), bl.begin() + static_cast<std::ptrdiff_t>(lslots[pid].size()), bl.end());
        }
        lslots[h.id] = ls;
        results.push_back(h.id);
      } catch (const kv::CacheError& e) {
        err = static_cast<int>(e.kind());
      }
    } else {
      kind = "release";
      std::uint64_t id;
      if (!released.empty() && rng.next_int(0, 9) == 0) {
        id = released[static_cast<std::size_t>(rng.next_int(0, static_cast<int>(released.size()) - 1))];
      } else {
        id = pick();
      }
      args.push_back(id);
      try {
        store.release(kv::SequenceHandle{id, lens[id]});
        live.erase(id);
        released.push_back(id);
      } catch (const kv::CacheError& e) {
        err = static_cast<int>(e.kind());
      }
    }
    auto st = store.stats();
    std::printf("{\"op\":\"%s\",", kind.c_str());
    put_vec("args", args);
    std::printf(",\"n\":%d,", n);
    put_vec("tokens", toks);
    std::printf(",");
    put_vec("results", results);
    std::printf(",\"error\":%d,\"logical\":%zu,\"live\":%zu,\"bytes_copied\":%zu,\"resolved\":[", err,
                st.logical_tokens_reachable, st.live_handles, st.bytes_copied_on_last_op);
    for (std::size_t i = 0; i < results.size(); ++i) {
      if (i) std::printf(",");
      emit_resolve(results[i]);
    }
    std::printf("]}\n");
  }
  std::printf("{\"final\":[");
  bool first = true;
  for (auto& [id, seq] : live) {
    if (!first) std::printf(",");
    first = false;
    emit_resolve(id);
  }
  std::printf("]}\n");
  return 0;
}

// ---------------------------------------------------------------------------
// toy goldens
// ---------------------------------------------------------------------------
void emit_forward(const std::string& name, const toy::ToyModelConfig& cfg, const std::string& text) {
  toy::ToyModel model(cfg);
  tok::Tokenizer tz;
  auto traj = grammar::parse_text(text);
  dag::TrainingBatch batch = dag::build_training_batch(traj, tz);
  auto fwd = model.forward(batch);
  std::printf("{\"kind\":\"forward\",\"name\":\"%s\",\"layers\":%d,\"heads\":%d,\"model_dim\":%d,\"vocab\":%d,"
              "\"seed\":%" PRIu64 ",\"init\":%.17g,\"rope\":%.17g,",
              name.c_str(), cfg.layers, cfg.heads, cfg.model_dim, cfg.vocab_size, cfg.seed, cfg.init_range,
              cfg.rope_base);
  put_vec("tokens", batch.token_ids);
  std::printf(",");
  put_vec("positions", batch.positions);
  std::printf(",");
  put_vec("logits", fwd.logits);
  std::printf(",\"loss\":%.17g}\n", model.loss(batch));
}

void emit_step(const std::string& name, const toy::ToyModelConfig& cfg, int ctx_len, int token, int pos,
               std::uint64_t seed) {
  toy::ToyModel model(cfg);
  synth::Rng rng(seed);
  std::vector<double> ctx(static_cast<std::size_t>(ctx_len) * static_cast<std::size_t>(cfg.kv_doubles_per_token()));
  for (auto& x : ctx) x = rng.next_symmetric(1.0);
  auto out = model.step(ctx, static_cast<std::size_t>(ctx_len), token, pos);
  std::printf("{\"kind\":\"step\",\"name\":\"%s\",\"layers\":%d,\"heads\":%d,\"model_dim\":%d,\"vocab\":%d,"
              "\"seed\":%" PRIu64 ",\"init\":%.17g,\"rope\":%.17g,\"ctx_len\":%d,\"token\":%d,\"pos\":%d,"
              "\"ctx_seed\":%" PRIu64 ",",
              name.c_str(), cfg.layers, cfg.heads, cfg.model_dim, cfg.vocab_size, cfg.seed, cfg.init_range,
              cfg.rope_base, ctx_len, token, pos, seed);
  put_vec("logits", out.logits);
  std::printf(",");
  put_vec("kv", out.kv);
  std::printf("}\n");
}

std::string c1_text(int prompt_words, int path_words, int concl_words) {
  synth::Rng rng(0);
  std::string s = synth::random_sequential_text(rng, prompt_words);
  s += " <Parallel> <Goal> <Outline> 1: first </Outline> <Outline> 2: second </Outline> </Goal> <Path> 1: ";
  s += synth::random_sequential_text(rng, path_words);
  s += " </Path> <Path> 2: ";
  s += synth::random_sequential_text(rng, path_words);
  s += " </Path> <Conclusion> ";
  s += synth::random_sequential_text(rng, concl_words);
  s += " </Conclusion> </Parallel>";
  return s;
}

void emit_forced(const std::string& name, const toy::ToyModelConfig& cfg, const std::string& text) {
  toy::ToyModel model(cfg);
  tok::Tokenizer tz;
  auto traj = grammar::parse_text(text);
  auto sm = engine::ScriptedModel::from_trajectory(traj, tz);
  engine::RunOptions opt;
  opt.record_logits = true;
  auto rep = engine::run_forced(sm, model, tz, opt);
  std::printf("{\"kind\":\"forced\",\"name\":\"%s\",\"status\":%d,\"total\":%zu,\"critical\":%zu,"
              "\"max_merge_bytes\":%zu,\"text\":\"%s\",",
              name.c_str(), static_cast<int>(rep.status), rep.total_tokens, rep.sequential_length,
              rep.max_merge_bytes_copied, json_escape(text).c_str());
  std::vector<double> flat;
  for (const auto& row : rep.logits_by_source) flat.insert(flat.end(), row.begin(), row.end());
  put_vec("logits", flat);
  std::printf("}\n");
}

int mode_toy() {
  toy::ToyModelConfig small;  // SPEC defaults: 2 layers, 2 heads, d=32, vocab 256
  const char* t1 =
      "plan <Parallel> <Goal> <Outline> 1: a </Outline> <Outline> 2: b </Outline> </Goal> "
      "<Path> 1: x1 x2 </Path> <Path> 2: y1 y2 y3 </Path> "
      "<Conclusion> done </Conclusion> </Parallel> end";
  emit_forward("t1_small", small, t1);
  toy::ToyModelConfig c1;
  c1.layers = 2;
  c1.heads = 4;
  c1.model_dim = 256;
  c1.vocab_size = 256;
  emit_forward("t1_c1", c1, t1);
  emit_step("step_small", small, 37, 123, 41, 7);
  emit_step("step_c1", c1, 64, 300, 1000, 8);
  emit_step("step_c1_empty", c1, 0, 5, 0, 9);
  emit_forced("forced_t1_small", small, t1);
  emit_forced("forced_c1_mini", c1, c1_text(48, 12, 6));
  return 0;
}

// engine::run_free (greedy, engine.cpp:941-950) of the C1 toy model after a seeded prompt: status,
// failure detail and every emitted token (Decode / Prefill events with the token's id).
void emit_free(const char* name, const toy::ToyModelConfig& cfg, int prompt_words, std::uint64_t seed) {
  toy::ToyModel model(cfg);
  synth::Rng rng(seed);
  const std::string text = synth::random_sequential_text(rng, prompt_words);
  tok::Tokenizer tz;
  auto prompt = tz.tokenize(text);
  engine::RunOptions opt;
  auto rep = engine::run_free(model, tz, prompt, opt);
  std::vector<int> prompt_ids, steps, lanes, kinds, ids;
  for (const auto& t : prompt) prompt_ids.push_back(t.id);
  for (const auto& e : rep.events) {
    if (e.kind != engine::EventKind::Decode && e.kind != engine::EventKind::Prefill) continue;
    steps.push_back(static_cast<int>(e.step));
    lanes.push_back(e.lane);
    kinds.push_back(e.kind == engine::EventKind::Decode ? 0 : 1);
    // token_from_id (engine.cpp:584-597): vocab text for known ids, "tok<id>" beyond the vocabulary
    auto known = tz.vocab().lookup(e.token);
    ids.push_back(known ? *known : std::stoi(e.token.substr(3)));
  }
  std::printf("{\"kind\":\"free\",\"name\":\"%s\",\"layers\":%d,\"heads\":%d,\"model_dim\":%d,\"vocab\":%d,"
              "\"seed\":%llu,\"init\":%.17g,\"rope\":%.17g,\"status\":%d,\"failure\":%d,\"detail\":\"%s\","
              "\"wall\":%.17g,",
              name, cfg.layers, cfg.heads, cfg.model_dim, cfg.vocab_size, (unsigned long long)cfg.seed, cfg.init_range,
              cfg.rope_base, static_cast<int>(rep.status), static_cast<int>(rep.failure), rep.failure_detail.c_str(),
              rep.wall_units);
  put_vec("prompt", prompt_ids);
  std::printf(",");
  put_vec("steps", steps);
  std::printf(",");
  put_vec("lanes", lanes);
  std::printf(",");
  put_vec("kinds", kinds);
  std::printf(",");
  put_vec("tokens", ids);
  std::printf("}\n");
}

int mode_free() {
  toy::ToyModelConfig c1;
  c1.layers = 2;
  c1.heads = 4;
  c1.model_dim = 256;
  c1.vocab_size = 256;
  emit_free("free_c1", c1, 512, 0);
  toy::ToyModelConfig small;
  emit_free("free_small", small, 64, 3);
  return 0;
}

int mode_forced_bench(int prompt_words, int path_words, int reps) {
  toy::ToyModelConfig c1;
  c1.layers = 2;
  c1.heads = 4;
  c1.model_dim = 256;
  c1.vocab_size = 256;
  toy::ToyModel model(c1);
  std::string text = c1_text(prompt_words, path_words, 32);
  double best = 1e30;
  std::size_t total = 0;
  for (int r = 0; r < reps; ++r) {
    tok::Tokenizer tz;
    auto traj = grammar::parse_text(text);
    auto sm = engine::ScriptedModel::from_trajectory(traj, tz);
    engine::RunOptions opt;
    opt.record_events = false;
    auto t0 = std::chrono::steady_clock::now();
    auto rep = engine::run_forced(sm, model, tz, opt);
    auto t1 = std::chrono::steady_clock::now();
    best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
    total = rep.total_tokens;
    if (rep.status != engine::RunStatus::Done) {
      std::fprintf(stderr, "run_forced failed: %s\n", rep.failure_detail.c_str());
      return 2;
    }
  }
  std::printf("{\"kind\":\"forced_bench\",\"tokens\":%zu,\"seconds\":%.6f,\"tokens_per_s\":%.3f}\n", total, best,
              static_cast<double>(total) / best);
  return 0;
}

// The reference's own decode path for BASELINE configs[1] (engine.cpp:599-607: resolve_payloads of
// the lane's context + ToyModel::step), one layer of Qwen2.5-32B attention shape (40 heads x 128;
// the reference has no GQA, so K/V per token are 40 heads wide), 4096-token shared prefix forked
// into 8 branches of 1023 tokens, timed on `threads` host threads (one branch per thread;
// RadixStore resolution is read-only and ToyModel::step is const).
// step() also runs the QKV/O projections and the MLP, which are not part of the attention path,
// so each sample also times step() with an empty context and reports the difference.
// threads lanes decode in parallel; with steps >= 0 every thread runs exactly warmup + steps
// branch-token decodes (a bench "step" = one token per thread) and only the last `steps` are timed,
// else each runs for `seconds`.
int mode_decode_bench(int threads, double seconds, int steps = -1, int warmup = 0) {
  toy::ToyModelConfig cfg;
  cfg.layers = 1;
  cfg.heads = 40;
  cfg.model_dim = 5120;
  cfg.vocab_size = 256;
  toy::ToyModel model(cfg);
  const std::size_t rec = static_cast<std::size_t>(cfg.kv_doubles_per_token()) * sizeof(double);
  kv::RadixStore store(rec, 1u << 16);
  synth::Rng rng(0);
  auto payload = [&](std::size_t n) {
    std::vector<double> d(n * cfg.kv_doubles_per_token());
    for (auto& x : d) x = rng.next_symmetric(1.0);
    std::vector<std::byte> b(d.size() * sizeof(double));
    std::memcpy(b.data(), d.data(), b.size());
    return b;
  };
  auto ids = [](std::size_t n, int base) {
    std::vector<kv::TokenId> t(n);
    for (std::size_t i = 0; i < n; ++i) t[i] = 10 + static_cast<int>((base + i) % 240);
    return t;
  };
  const std::size_t prefix = 4096, blen = 1023;
  const int nb = 8;
  auto root = store.create();
  auto pfx_ids = ids(prefix, 0);
  auto pfx = store.extend(root, pfx_ids, payload(prefix));
  auto kids = store.fork(pfx, nb);
  std::vector<kv::SequenceHandle> br;
  for (int b = 0; b < nb; ++b) {
    auto bi = ids(blen, 1000 * (b + 1));
    br.push_back(store.extend(kids[b], bi, payload(blen)));
  }
  std::vector<double> t_full(threads, 0.0), t_empty(threads, 0.0);
  std::vector<int> reps(threads, 0);
  const auto start = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      const auto& h = br[t % nb];
      const int pos = static_cast<int>(prefix + blen);
      for (int it = 0;; ++it) {
        if (steps >= 0 ? it >= warmup + steps
                       : (std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count() >= seconds &&
                          reps[t] > 0))
          break;
        auto a = std::chrono::steady_clock::now();
        auto ctx = store.resolve_payloads(h);
        auto out = model.step(std::span<const double>(reinterpret_cast<const double*>(ctx.data()), ctx.size() / sizeof(double)),
                              h.length, 13, pos);
        auto b = std::chrono::steady_clock::now();
        auto out0 = model.step(std::span<const double>(), 0, 13, pos);
        auto c = std::chrono::steady_clock::now();
        if (steps >= 0 && it < warmup) continue;
        t_full[t] += std::chrono::duration<double>(b - a).count();
        t_empty[t] += std::chrono::duration<double>(c - b).count();
        reps[t] += 1;
        if (out.logits.empty() || out0.logits.empty()) std::abort();
      }
    });
  for (auto& th : pool) th.join();
  double full = 0, empty = 0;
  int n = 0;
  for (int t = 0; t < threads; ++t) {
    full += t_full[t];
    empty += t_empty[t];
    n += reps[t];
  }
  const double per_full = full / n, per_attn = (full - empty) / n;
  std::printf("{\"kind\":\"decode_bench\",\"threads\":%d,\"steps\":%d,\"ctx\":%zu,\"s_per_token_full\":%.6f,"
              "\"s_per_token_attention\":%.6f,\"tokens_per_s_full\":%.4f,\"tokens_per_s_attention\":%.4f}\n",
              threads, n, prefix + blen, per_full, per_attn, threads / per_full, threads / per_attn);
  return 0;
}

// C5 op log on the reference RadixStore.  Stops after the round in which `budget_s` seconds have
// elapsed (its bookkeeping grows quadratically with the rounds) and prints the
// per-round op times so the caller can extrapolate the remaining rounds.
int mode_c5(int rounds, std::size_t rec, double budget_s = 1e30) {
  using clk = std::chrono::steady_clock;
  kv::RadixStore store(rec, 1u << 20);
  std::vector<std::byte> zeros(rec * 4096);
  auto ids = [](std::size_t n, int base) {
    std::vector<kv::TokenId> t(n);
    for (std::size_t i = 0; i < n; ++i) t[i] = 10 + static_cast<int>((base + 7 * i) % 240);
    return t;
  };
  auto us = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
  auto root = store.create();
  auto cur = store.extend(root, ids(4096, 0), std::span<const std::byte>(zeros.data(), rec * 4096));
  store.release(root);
  double t_fork = 0, t_ext = 0, t_merge = 0, t_rel = 0, t_red = 0;
  int n_ext = 0, n_rel = 0, done = 0;
  std::vector<double> round_us;
  const auto t_start = clk::now();
  for (int r = 0; r < rounds; ++r) {
    const auto r0 = clk::now();
    auto a = clk::now();
    auto kids = store.fork(cur, 128);
    auto b = clk::now();
    t_fork += us(a, b);
    std::vector<kv::SequenceHandle> ext;
    for (int k = 0; k < 128; ++k) {
      auto c = clk::now();
      ext.push_back(store.extend(kids[k], ids(64, 1000 * (r + 1) + 13 * k), std::span<const std::byte>(zeros.data(), rec * 64)));
      t_ext += us(c, clk::now());
      ++n_ext;
    }
    auto d = clk::now();
    auto m = store.merge(cur, ext);
    auto e = clk::now();
    t_merge += us(d, e);
    auto f = clk::now();
    store.release(cur);
    for (auto& h : kids) store.release(h);
    for (auto& h : ext) store.release(h);
    t_rel += us(f, clk::now());
    n_rel += 1 + 256;
    auto g = clk::now();
    auto nm = store.extend(m, ids(16, 7), std::span<const std::byte>(zeros.data(), rec * 16));
    store.release(m);
    t_red += us(g, clk::now());
    cur = nm;
    round_us.push_back(us(r0, clk::now()));
    ++done;
    if (std::chrono::duration<double>(clk::now() - t_start).count() > budget_s) break;
  }
  rounds = done;
  std::string per_round = "[";
  for (std::size_t i = 0; i < round_us.size(); ++i) per_round += (i ? "," : "") + std::to_string(round_us[i]);
  per_round += "]";
  std::printf("{\"kind\":\"c5\",\"rounds\":%d,\"final_len\":%zu,\"fork128_us\":%.3f,\"extend64_us\":%.3f,"
              "\"merge128_us\":%.3f,\"release_us\":%.3f,\"reduce_extend16_us\":%.3f,\"round_us\":%s}\n",
              rounds, cur.length, t_fork / rounds, t_ext / n_ext, t_merge / rounds, t_rel / n_rel, t_red / rounds,
              per_round.c_str());
  store.release(cur);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: refdrv dag <fixtures>|kv <seed> <ops> <rec>|toy|forced <words> <pathw> <reps>\n");
    return 1;
  }
  std::string mode = argv[1];
  if (mode == "dag" && argc >= 3) return mode_dag(argv[2]);
  if (mode == "batch" && argc >= 3) return mode_batch(argv[2]);
  if (mode == "kv" && argc >= 5)
    return mode_kv(std::stoull(argv[2]), std::stoi(argv[3]), static_cast<std::size_t>(std::stoul(argv[4])));
  if (mode == "toy") return mode_toy();
  if (mode == "free") return mode_free();
  if (mode == "forced" && argc >= 5) return mode_forced_bench(std::stoi(argv[2]), std::stoi(argv[3]), std::stoi(argv[4]));
  if (mode == "decode" && argc >= 6)
    return mode_decode_bench(std::stoi(argv[2]), std::stod(argv[3]), std::stoi(argv[4]), std::stoi(argv[5]));
  if (mode == "decode" && argc >= 4) return mode_decode_bench(std::stoi(argv[2]), std::stod(argv[3]));
  if (mode == "c5" && argc >= 5)
    return mode_c5(std::stoi(argv[2]), static_cast<std::size_t>(std::stoul(argv[3])), std::stod(argv[4]));
  if (mode == "c5" && argc >= 4) return mode_c5(std::stoi(argv[2]), static_cast<std::size_t>(std::stoul(argv[3])));
  std::fprintf(stderr, "bad arguments\n");
  return 1;
}
