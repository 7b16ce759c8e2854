#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY: compiles the reference's own translation units
# (/root/reference/proj/core/src/*.cpp, unmodified) with patched COPIES of its headers and the
# SPEC-following glue in oracle/ref_glue/ into oracle/_ref/tmg_ref_bench. Outputs only under
# oracle/_ref/ (git-ignored; it travels to the GPU box with the snapshot). Skips quietly when the
# reference is absent (the GPU box).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF=/root/reference/proj/core
OUT="$HERE/_ref"
[ -d "$REF" ] || { echo "build_ref: $REF absent, skipping"; exit 0; }
JSON_INC="$(python3 - <<'PY'
import glob, os, sys
for p in glob.glob(sys.prefix + "/lib/python3*/site-packages/include/cudnn_frontend/thirdparty"):
    if os.path.exists(os.path.join(p, "nlohmann", "json.hpp")):
        print(p); break
PY
)"
[ -n "$JSON_INC" ] || { echo "build_ref: vendored nlohmann/json.hpp not found"; exit 1; }
mkdir -p "$OUT/include" "$OUT/obj"
rm -rf "$OUT/include/tmg"
cp -r "$REF/include/tmg" "$OUT/include/tmg"
python3 "$HERE/patch_ref_headers.py" "$OUT/include"
CXX="${CXX:-g++}"
FLAGS="-O2 -std=c++20 -pthread -I$OUT/include -I$JSON_INC"
pids=()
for src in "$REF"/src/*.cpp; do
  obj="$OUT/obj/$(basename "$src" .cpp).o"
  if [ ! -f "$obj" ] || [ "$src" -nt "$obj" ]; then
    $CXX $FLAGS -c "$src" -o "$obj" & pids+=($!)
  fi
done
for p in "${pids[@]}"; do wait "$p"; done
$CXX $FLAGS "$HERE/ref_glue/tmg_ref_bench.cpp" "$OUT"/obj/*.o -o "$OUT/tmg_ref_bench"
echo "build_ref: $OUT/tmg_ref_bench"
# the reference-side binding of the drop-in against the built libtmgx.so
LIB="$HERE/../paper_1604_07163_b200"
if [ -f "$LIB/libtmgx.so" ]; then
  $CXX $FLAGS -I"$HERE/../include" "$HERE/ref_glue/tmg_ref_gpupc.cpp" "$OUT"/obj/*.o -L"$LIB" -ltmgx \
    -Wl,-rpath,'$ORIGIN/../../paper_1604_07163_b200' -ldl -lrt -o "$OUT/tmg_ref_gpupc"
  echo "build_ref: $OUT/tmg_ref_gpupc"
  $CXX $FLAGS -I"$HERE/../include" "$HERE/ref_glue/tmg_ref_gpupc.cpp" "$OUT"/obj/*.o -L"$LIB" -l:libtmgx_parity.so \
    -Wl,-rpath,'$ORIGIN/../../paper_1604_07163_b200' -ldl -lrt -o "$OUT/tmg_ref_gpupc_parity"
  echo "build_ref: $OUT/tmg_ref_gpupc_parity"
fi
