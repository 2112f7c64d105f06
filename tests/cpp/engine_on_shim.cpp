// The reference's engine::run_forced (engine.cpp:928-939), compiled from /root/reference against the
// drop-in headers in tests/cpp/refswap (multiverse::kv -> the device paged store, multiverse::toy -> the
// device toy model), driving the same forced streams as tests/golden/toy.jsonl.gz.  Prints one JSON line
// per run with the logits by source index; tests/test_refswap_gpu.py compares them with the golden
// logits the unmodified reference produced.  Test infrastructure (built by tests/cpp/build_refswap.sh).
#include <cstdio>
#include <string>

#include "multiverse/engine.hpp"
#include "multiverse/grammar.hpp"
#include "multiverse/synth.hpp"
#include "multiverse/tokenizer.hpp"

using namespace multiverse;

static std::string c1_text(int prompt_words, int path_words, int concl_words) {  // oracle/refdrv.cpp c1_text
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

static void run(const char* name, const toy::ToyModelConfig& cfg, const std::string& text) {
  toy::ToyModel model(cfg);
  tok::Tokenizer tz;
  auto sm = engine::ScriptedModel::from_trajectory(grammar::parse_text(text), tz);
  engine::RunOptions opt;
  opt.record_logits = true;
  auto rep = engine::run_forced(sm, model, tz, opt);
  std::printf("{\"name\":\"%s\",\"status\":%d,\"total\":%zu,\"critical\":%zu,\"max_merge_bytes\":%zu,\"logits\":[",
              name, static_cast<int>(rep.status), rep.total_tokens, rep.sequential_length,
              rep.max_merge_bytes_copied);
  bool first = true;
  for (const auto& row : rep.logits_by_source)
    for (double x : row) {
      std::printf(first ? "%.9g" : ",%.9g", x);
      first = false;
    }
  std::printf("]}\n");
}

int main() {
  toy::ToyModelConfig small;
  run("forced_t1_small", small,
      "plan <Parallel> <Goal> <Outline> 1: a </Outline> <Outline> 2: b </Outline> </Goal> "
      "<Path> 1: x1 x2 </Path> <Path> 2: y1 y2 y3 </Path> <Conclusion> done </Conclusion> </Parallel> end");
  toy::ToyModelConfig c1;
  c1.layers = 2;
  c1.heads = 4;
  c1.model_dim = 256;
  c1.vocab_size = 256;
  run("forced_c1_mini", c1, c1_text(48, 12, 6));
  return 0;
}
