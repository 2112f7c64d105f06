#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY. Builds tests/cpp/_build/engine_on_shim: the reference's OWN engine.cpp
# (with grammar / dag / tokenizer / synth, the parts of proj/core this path does not replace),
# compiled from the sources where they lie under /root/reference against the drop-in headers in
# tests/cpp/refswap, which switch multiverse::kv and multiverse::toy to include/multiverse_b200.hpp
# (the device paged store and toy model behind libmvb200.so).  The reference's kvcache.cpp and
# toy_model.cpp are NOT linked: the engine runs on this repo's implementation.  The two one-line
# reference fixes (BUG-1, BUG-2; oracle/ref_patch.py) are applied to a scratch copy.
# Output: tests/cpp/_build/ (git-ignored; travels to the GPU box with the snapshot).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REPO="$(cd "$HERE/../.." && pwd)"
REF="${MV_REFERENCE:-/root/reference/proj/core}"
OUT="$HERE/_build"
if [ ! -d "$REF" ]; then echo "reference not present at $REF; skipping the engine-on-shim build"; exit 0; fi
mkdir -p "$OUT"
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF/include" "$TMP/include"
mkdir -p "$TMP/src"
for f in dag grammar tokenizer synth engine; do cp "$REF/src/$f.cpp" "$TMP/src/"; done
python3 "$REPO/oracle/ref_patch.py" "$TMP" > /dev/null
CXX=${CXX:-g++}
# refswap FIRST: engine.hpp's #include "multiverse/kvcache.hpp" / "multiverse/toy_model.hpp" resolve here
FLAGS="-std=c++20 -O2 -I$HERE/refswap -I$TMP/include -I$REPO/include -I/usr/local/cuda/include"
objs=()
for f in dag grammar tokenizer synth engine; do
  $CXX $FLAGS -c "$TMP/src/$f.cpp" -o "$TMP/$f.o" &
  objs+=("$TMP/$f.o")
done
wait
$CXX $FLAGS "$HERE/engine_on_shim.cpp" "${objs[@]}" -o "$OUT/engine_on_shim" \
  -L"$REPO/paper_2506_09991_b200" -lmvb200 -L/usr/local/cuda/lib64 -lcudart \
  -Wl,-rpath,'$ORIGIN/../../../paper_2506_09991_b200' -Wl,-rpath,/usr/local/cuda/lib64
echo "built $OUT/engine_on_shim"
