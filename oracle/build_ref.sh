#!/usr/bin/env bash
# Builds the REFERENCE CPU implementation (oracle/_ref/libpintswe_ref.so) from the sources where
# they lie under /root/reference/proj/src, plus the FFTW3-API shim and the extern "C" harness in
# oracle/ref_build/. Test/baseline infrastructure only (see oracle/README.md).
#   -include algorithm : proj/include/pintswe/field.hpp:105 uses std::max({..}) without <algorithm>
#   io.cpp / runner.cpp / cases.cpp are not compiled (need nlohmann/json / are off the hot path).
# -march=x86-64-v3 (AVX2) instead of -march=native so the .so runs on the GPU box's host, and
# -ffp-contract=off: the reference's own CMake Release build (proj/CMakeLists.txt, no -march)
# targets baseline x86-64, which has no FMA, so its arithmetic never contracts a*b+c. With
# contraction on, g++ fuses the Legendre recurrence / H-table products and the T511 divergence
# tendency moves from 2.8e-12 to 1.2e-11 away from the exact discrete operator (oracle/precise.py).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${PSWE_REFERENCE:-/root/reference}/proj"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then echo "reference sources not found at $REF; skipping oracle/_ref build"; exit 0; fi
mkdir -p "$OUT"
SRCS="gauss legendre transform reference swe quadrature sdc multilevel pfasst analysis"
FILES=""
for s in $SRCS; do FILES="$FILES $REF/src/$s.cpp"; done
# io.cpp needs nlohmann/json (vendor/ is absent, proj/.gitignore:2); use the copy in the image if any
JSON_DIR=/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
IOFLAGS=""
if [ -f "$JSON_DIR/json.hpp" ]; then IOFLAGS="-I$JSON_DIR -DPSWE_REF_WITH_IO"; FILES="$FILES $REF/src/io.cpp"; fi
g++ -std=c++20 -O3 -march=x86-64-v3 -ffp-contract=off -fopenmp -fPIC -shared -include algorithm \
    -I"$REF/include" -I"$HERE/ref_build" $IOFLAGS $FILES "$HERE/ref_build/ref_capi.cpp" \
    -o "$OUT/libpintswe_ref.so.tmp" -lpthread
mv "$OUT/libpintswe_ref.so.tmp" "$OUT/libpintswe_ref.so"
echo "built $OUT/libpintswe_ref.so"

# GpuImexOde drop-in: the reference's sdc/multilevel/pfasst sources + the adapter over libpswe.so
PSWE_LIB_DIR="$(cd "$HERE/.." && pwd)/paper_1904_05988_b200"
if [ -f "$PSWE_LIB_DIR/libpswe.so" ]; then
  g++ -std=c++20 -O3 -march=x86-64-v3 -ffp-contract=off -fopenmp -fPIC -shared -include algorithm \
      -I"$REF/include" -I"$HERE/ref_build" -I"$HERE/../include" $IOFLAGS \
      $FILES "$HERE/ref_build/gpu_imexode.cpp" -o "$OUT/libpintswe_gpu.so.tmp" \
      -L"$PSWE_LIB_DIR" -lpswe -Wl,-rpath,'$ORIGIN/../../paper_1904_05988_b200' -lpthread
  mv "$OUT/libpintswe_gpu.so.tmp" "$OUT/libpintswe_gpu.so"
  echo "built $OUT/libpintswe_gpu.so"
fi
