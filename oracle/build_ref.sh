#!/usr/bin/env bash
# Build oracle/_ref/libtierq_ref.so from the REFERENCE sources where they lie
# under /root/reference/proj (read-only; never copied into this repo) plus
# oracle/ref_shim.cpp.  Only the columnar substrate exists there:
# common.cpp and src/columnar/*.cpp compile standalone with g++ -std=c++20.
# Output goes only to oracle/_ref/ (git-ignored, shipped to the GPU box).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${TQ_REFERENCE_ROOT:-/root/reference}/proj"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "build_ref: reference sources not present at $REF; keeping prebuilt $OUT" >&2
  exit 0
fi
mkdir -p "$OUT"
g++ -std=c++20 -O2 -fPIC -shared -Wall -Wextra -pthread \
  -I"$REF/include" \
  "$REF/src/common.cpp" \
  "$REF/src/columnar/types.cpp" \
  "$REF/src/columnar/transform.cpp" \
  "$REF/src/columnar/pool.cpp" \
  "$REF/src/columnar/chunked.cpp" \
  "$REF/src/columnar/serde.cpp" \
  "$HERE/ref_shim.cpp" \
  -o "$OUT/libtierq_ref.so.tmp"
mv "$OUT/libtierq_ref.so.tmp" "$OUT/libtierq_ref.so"
echo "build_ref: built $OUT/libtierq_ref.so"

# The C++ binding of INTEGRATION.md §2-3, compiled against the reference's
# headers + columnar sources and libtq_gpu.so's C-ABI (test infrastructure;
# needs a GPU to run: tests/test_boundary.py, -m gpu).
LIB="$HERE/../paper_2508_05029_b200"
if [ -f "$LIB/libtq_gpu.so" ]; then
  g++ -std=c++20 -O2 -Wall -Wextra -pthread \
    -I"$REF/include" -I"$HERE/../include" \
    "$HERE/boundary_test.cpp" \
    "$REF/src/common.cpp" \
    "$REF/src/columnar/types.cpp" \
    "$REF/src/columnar/transform.cpp" \
    -L"$LIB" -ltq_gpu -Wl,-rpath,'$ORIGIN/../../paper_2508_05029_b200' \
    -o "$OUT/boundary_test.tmp"
  mv "$OUT/boundary_test.tmp" "$OUT/boundary_test"
  echo "build_ref: built $OUT/boundary_test"
fi
