#!/usr/bin/env bash
# Compiles the reference-side binding (tests/cabi/gpu_pipeline_harness.cpp + harness_main.cpp)
# against the UNMODIFIED reference headers (/root/reference/proj/include, read in place) and links
# it with the reference library built by build_ref.sh plus libpsg.so. Output: oracle/_ref/
# (git-ignored, travels to the GPU box, where /root/reference does not exist).
set -euo pipefail
REF=${REF:-/root/reference/proj}
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(dirname "$HERE")"
OUT="$HERE/_ref"
JSON_DIR=${JSON_DIR:-/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann}
if [ ! -d "$REF/include" ] || [ ! -f "$OUT/libpystachio_ref.a" ]; then echo "reference not present; skipping" >&2; exit 0; fi
LIB="$ROOT/paper_2512_02862_b200"
g++ -std=c++20 -O2 -pthread -I"$REF/include" -I"$JSON_DIR" -I"$ROOT/include" -I"$ROOT/tests/cabi" \
  "$ROOT/tests/cabi/gpu_pipeline_harness.cpp" "$ROOT/tests/cabi/harness_main.cpp" \
  -L"$OUT" -lpystachio_ref -L"$LIB" -lpsg -Wl,-rpath,"$LIB" -lz -o "$OUT/gpu_pipeline_harness"
echo "built $OUT/gpu_pipeline_harness"
