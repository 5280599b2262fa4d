#!/usr/bin/env bash
# Build the C++ drop-in test programs into tests/cpp/_build (git-ignored, travel to the GPU box).
set -e
HERE=$(cd "$(dirname "$0")" && pwd); ROOT=$(cd "$HERE/../.." && pwd)
OUT=$HERE/_build; mkdir -p "$OUT"
LIB=$ROOT/paper_1204_5072_b200/_lib
g++ -std=c++17 -O2 -Wall -Wextra -I"$ROOT/include" "$HERE/dropin_test.cpp" -L"$LIB" -llfg \
    -Wl,-rpath,'$ORIGIN/../../../paper_1204_5072_b200/_lib' -o "$OUT/dropin_standalone"
REF=${REF:-/root/reference}
if [ -d "$REF/proj/include" ] && [ -f "$ROOT/oracle/_ref/liblfref.so" ]; then
  g++ -std=c++20 -O2 -Wall -Wextra -include string -DLF_WITH_REFERENCE -I"$ROOT/include" -I"$REF/proj/include" \
      "$HERE/dropin_test.cpp" -L"$LIB" -llfg -L"$ROOT/oracle/_ref" -llfref \
      -Wl,-rpath,'$ORIGIN/../../../paper_1204_5072_b200/_lib:$ORIGIN/../../../oracle/_ref' -o "$OUT/dropin_reference"
fi
# Link-level drop-in: the reference's own headers and sources, with kpz.cpp and
# kmc.cpp replaced by dropin/lf_gpu_link.cpp (built here; the binary travels).
if [ -d "$REF/proj/src" ]; then
  g++ -std=c++20 -O2 -Wall -Wextra -include string -I"$ROOT/include" -I"$REF/proj/include" \
      "$HERE/linkdrop_test.cpp" "$ROOT/dropin/lf_gpu_link.cpp" \
      "$REF/proj/src/lattice.cpp" "$REF/proj/src/rng.cpp" -L"$LIB" -llfg \
      -Wl,-rpath,'$ORIGIN/../../../paper_1204_5072_b200/_lib' -o "$OUT/linkdrop_reference"
fi
