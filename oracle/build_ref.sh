#!/usr/bin/env bash
# Test infrastructure only: compiles the UNMODIFIED reference engine from its sources under
# /root/reference/proj (read in place, never copied) into oracle/_ref/, plus our own driver
# (oracle/ref_driver.cpp) that calls the reference's public API. Outputs go to oracle/_ref/ only
# (git-ignored; travels to the GPU box with gpurun snapshots so bench.py --impl reference can run).
#
# The reference's include `<json.hpp>` is satisfied by the nlohmann/json 3.x single header that
# ships inside the venv (cudnn_frontend/thirdparty); doctest/CLI11 are not needed for this target.
set -euo pipefail
REF=${REF:-/root/reference/proj}
HERE="$(cd "$(dirname "$0")" && pwd)"
OUT="$HERE/_ref"
JSON_DIR=${JSON_DIR:-/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann}
if [ ! -d "$REF/src" ]; then echo "reference sources not present at $REF; skipping" >&2; exit 0; fi
mkdir -p "$OUT/obj"
CXX=${CXX:-g++}
FLAGS="-std=c++20 -O2 -pthread -I$REF/include -I$JSON_DIR"
pids=()
for f in "$REF"/src/*.cpp; do
  o="$OUT/obj/$(basename "$f" .cpp).o"
  if [ ! -f "$o" ] || [ "$f" -nt "$o" ]; then
    $CXX $FLAGS -c "$f" -o "$o" & pids+=($!)
  fi
done
for p in "${pids[@]}"; do wait "$p"; done
rm -f "$OUT/libpystachio_ref.a"
ar rcs "$OUT/libpystachio_ref.a" "$OUT"/obj/*.o
$CXX $FLAGS "$HERE/ref_driver.cpp" -L"$OUT" -lpystachio_ref -lz -o "$OUT/ref_driver"
echo "built $OUT/ref_driver"
