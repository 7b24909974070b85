#!/bin/bash
# Build an A/B variant of libpswe with extra nvcc flags: tools/build_variant.sh NAME "-DFLAG=1 ..."
# -> paper_1904_05988_b200/libpswe_NAME.so, loaded when PSWE_LIB_VARIANT=NAME (tuning only).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
make -s -j8 -C "$ROOT/paper_1904_05988_b200/csrc" OUT="$ROOT/paper_1904_05988_b200/libpswe_$1.so" \
    OBJDIR="$ROOT/build/pswe_$1" EXTRA_NVFLAGS="$2" 2>&1 | grep -E "error" || true
