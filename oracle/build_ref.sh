#!/usr/bin/env bash
# Builds the REFERENCE CPU implementation (oracle/_ref/libpintswe_ref.so) from the sources where
# they lie under /root/reference/proj/src, plus the FFTW3-API shim and the extern "C" harness in
# oracle/ref_build/. Test/baseline infrastructure only (see oracle/README.md).
#   -include algorithm : proj/include/pintswe/field.hpp:105 uses std::max({..}) without <algorithm>
#   io.cpp / runner.cpp / cases.cpp are not compiled (need nlohmann/json / are off the hot path).
# -march=x86-64-v3 (AVX2+FMA) instead of -march=native so the .so runs on the GPU box's host.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${PSWE_REFERENCE:-/root/reference}/proj"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then echo "reference sources not found at $REF; skipping oracle/_ref build"; exit 0; fi
mkdir -p "$OUT"
SRCS="gauss legendre transform reference swe quadrature sdc multilevel pfasst analysis"
FILES=""
for s in $SRCS; do FILES="$FILES $REF/src/$s.cpp"; done
g++ -std=c++20 -O3 -march=x86-64-v3 -fopenmp -fPIC -shared -include algorithm \
    -I"$REF/include" -I"$HERE/ref_build" $FILES "$HERE/ref_build/ref_capi.cpp" \
    -o "$OUT/libpintswe_ref.so.tmp" -lpthread
mv "$OUT/libpintswe_ref.so.tmp" "$OUT/libpintswe_ref.so"
echo "built $OUT/libpintswe_ref.so"
