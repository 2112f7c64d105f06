// TEST INFRASTRUCTURE ONLY (oracle/). Runs the reference's own per-lane tag interpreter
// (feed_interpreter, engine.cpp:323-415, with the BUG-2 fix of oracle/ref_patch.py) over event
// streams read from stdin, so the device interpreter (csrc/interp.cu) is pinned against the
// reference itself. Built by oracle/ref_build.sh from the patched scratch copy of engine.cpp,
// which this translation unit includes (the interpreter lives in an anonymous namespace there);
// nothing from the reference is copied into the repo.
//
// stdin:  one case per line: "<is_child> <n> e_0 ... e_{n-1}", e >= 0 a token id (ids 0..9 are
//         the tags in TagKind order, tokenizer.cpp:56-63), e == -2 the merge completion of
//         engine.cpp:793 (top frame -> AwaitConclusionTag), e == -1 an idle step (no call).
// stdout: per event "kind arg depth phase outlines in_outline after_outline" where kind is
//         InterpAction::Kind (0 None, 1 Spawn, 2 WorkerDone, 3 Violation), arg the spawn count;
//         a violation line is followed by "#<detail>". A merge with no open frame (undefined in
//         the reference: frames.back() on an empty vector) prints kind 3 and "#merge without an
//         open block" without touching the state.
#include "engine.cpp"  // the patched scratch copy (-I oracle/_ref/src/src)

#include <iostream>

namespace multiverse::engine {
void mv_drive_interp() {
  static const char* lit[] = {"<Parallel>", "</Parallel>", "<Goal>",  "</Goal>",       "<Outline>",
                              "</Outline>", "<Path>",      "</Path>", "<Conclusion>", "</Conclusion>"};
  int is_child, n;
  while (std::cin >> is_child >> n) {
    LaneRuntime lane;
    lane.parent = is_child ? 0 : -1;
    for (int i = 0; i < n; ++i) {
      int e;
      std::cin >> e;
      InterpAction a;
      if (e == -1) {
      } else if (e == -2) {
        if (lane.frames.empty()) {
          a.kind = InterpAction::Kind::Violation;
          a.detail = "merge without an open block";
        } else {
          lane.frames.back().phase = InterpFrame::Phase::AwaitConclusionTag;
        }
      } else {
        Token t;
        t.id = e;
        t.is_tag = e < 10;
        t.tag = t.is_tag ? static_cast<TagKind>(e) : TagKind::Text;
        t.text = t.is_tag ? lit[e] : "w" + std::to_string(e);
        a = feed_interpreter(lane, t);
      }
      int depth = static_cast<int>(lane.frames.size());
      const InterpFrame f = depth ? lane.frames.back() : InterpFrame{};
      std::cout << static_cast<int>(a.kind) << ' ' << a.spawn_count << ' ' << depth << ' '
                << static_cast<int>(f.phase) << ' ' << f.outlines << ' ' << f.in_outline << ' '
                << f.after_outline << '\n';
      if (a.kind == InterpAction::Kind::Violation) std::cout << '#' << a.detail << '\n';
    }
    std::cout << "end\n";
  }
}
}  // namespace multiverse::engine

int main() {
  multiverse::engine::mv_drive_interp();
  return 0;
}
