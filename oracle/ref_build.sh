#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY. Builds the patched reference core (oracle/_ref) from the
# sources where they lie under /root/reference. Outputs go only to oracle/_ref/
# (git-ignored). Nothing in the product links this.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${MV_REFERENCE:-/root/reference/proj/core}"
OUT="$HERE/_ref"
if [ ! -d "$REF" ]; then echo "reference not present at $REF; skipping _ref build"; exit 0; fi
rm -rf "$OUT/src"; mkdir -p "$OUT/src"
cp -r "$REF/include" "$OUT/src/include"
mkdir -p "$OUT/src/src"
for f in dag grammar kvcache synth tokenizer toy_model engine; do cp "$REF/src/$f.cpp" "$OUT/src/src/"; done
python3 "$HERE/ref_patch.py" "$OUT/src"
CXX=${CXX:-g++}
FLAGS="-std=c++20 -O2 -fPIC -I$OUT/src/include"
objs=()
for f in dag grammar kvcache synth tokenizer toy_model engine; do
  $CXX $FLAGS -c "$OUT/src/src/$f.cpp" -o "$OUT/$f.o" &
  objs+=("$OUT/$f.o")
done
wait
$CXX $FLAGS "$HERE/refdrv.cpp" "${objs[@]}" -o "$OUT/refdrv" -lpthread
# the reference's own per-lane tag interpreter (engine.cpp:323-415), for tests/golden/interp.jsonl.gz
$CXX $FLAGS -I"$OUT/src/src" "$HERE/interp_drv.cpp" "$OUT"/{dag,grammar,kvcache,synth,tokenizer,toy_model}.o \
  -o "$OUT/interp_drv"
rm -rf "$OUT/src"  # patched copies were build inputs only
echo "built $OUT/refdrv"
