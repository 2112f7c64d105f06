#!/usr/bin/env python3
"""TEST INFRASTRUCTURE ONLY (oracle/): applies the two one-line fixes documented in
SURVEY.md §0 to a scratch copy of the reference core under oracle/_ref/src.

Nothing here is shipped or measured; the patched copy lives only in the
git-ignored oracle/_ref/ build directory and is used to generate golden vectors
and, optionally, as the reference CPU baseline.

BUG-1 (core/src/dag.cpp:147 -> :160-162,:179,:183): `auto& info = dag_.blocks[..]`
       dangles after the nested visit_block reallocates dag_.blocks. Fix: re-index
       dag_.blocks[block_index] at every use after visit_nodes.
BUG-2 (core/src/engine.cpp:332-348): a fresh worker lane has no frames, so the
       injected <Path> falls into the `default: violation(...)` arm. Fix: accept
       <Path> on worker lanes (lane.parent >= 0).
"""
import pathlib
import sys

root = pathlib.Path(sys.argv[1])

dag = root / "src" / "dag.cpp"
s = dag.read_text()
anchor = "      visit_nodes(block.paths[k].nodes);\n"
assert anchor in s, "BUG-1 anchor not found"
head, tail = s.split(anchor, 1)
end = tail.index("  Tokenizer& tok_;")
body = tail[:end].replace("info.", "dag_.blocks[static_cast<std::size_t>(block_index)].")
s = head + anchor + body + tail[end:]
dag.write_text(s)

eng = root / "src" / "engine.cpp"
s = eng.read_text()
anchor = "      case TagKind::PathClose: {\n        if (lane.parent >= 0) {\n"
assert s.count(anchor) == 1, "BUG-2 anchor not found"
s = s.replace(anchor,
              "      case TagKind::PathOpen:\n        if (lane.parent >= 0) return none;\n"
              "        return violation(\"unexpected <Path> in sequential decode\");\n" + anchor)
eng.write_text(s)
print("patched", dag, eng)
