#!/usr/bin/env bash
# TEST INFRASTRUCTURE: compiles the UNMODIFIED reference library straight from
# its sources under /root/reference/proj (read-only; nothing is copied) plus
# oracle/ref_shim.cpp into oracle/_ref/libvoxref.so.  oracle/_ref/ is
# git-ignored but travels to the GPU box with the gpurun snapshot, where it is
# the CPU baseline / reference arm of bench.py and a parity checker in tests.
# Only the library core is needed (no CLI11 / nlohmann / doctest).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${VOXIN_REF:-/root/reference/proj}"
OUT="$HERE/_ref"
if [ ! -d "$REF/include/voxin" ]; then
  echo "build_ref: reference sources not found at $REF (expected on the GPU box: use the prebuilt _ref)" >&2
  exit 0
fi
mkdir -p "$OUT"
# x86-64-v3 (AVX2/FMA): runs on any current server host, including the GPU box
g++ -std=c++20 -O3 -march=x86-64-v3 -fPIC -shared -pthread \
  -I "$REF/include" \
  "$HERE/ref_shim.cpp" "$REF/src/parallel.cpp" "$REF/src/cost.cpp" \
  "$REF/src/planner.cpp" "$REF/src/netspec.cpp" \
  -o "$OUT/libvoxref.so.tmp"
mv "$OUT/libvoxref.so.tmp" "$OUT/libvoxref.so"
echo "built $OUT/libvoxref.so"
