#!/usr/bin/env bash
# Builds oracle/_ref/libtaskfmm_ref.so from the UNMODIFIED reference sources where
# they lie (/root/reference/proj/src/*.cpp), compiled directly with g++ (no CMake,
# no reference build system), against oracle/eigen_shim (our Eigen-surface shim
# over the image's OpenBLAS/LAPACK) plus oracle/ref_driver.cpp (our C ABI).
# Output goes only to oracle/_ref/ (git-ignored, travels to the GPU box with gpurun).
# Flags: -O3 without -march=native and with -ffp-contract=off so the reference's
# FP64 geometry (geometry.cpp:18-36, 76-91, 163-175) is plain IEEE (no FMA
# contraction); the B200 path reproduces those roundings explicitly.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${REF_ROOT:-/root/reference/proj}"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "build_ref: $REF not present; using prebuilt $OUT" >&2
  exit 0
fi
SCIPY_LIBS="$(python3 -c 'import scipy, os; print(os.path.join(os.path.dirname(scipy.__file__), os.pardir, "scipy.libs"))')"
SCIPY_LIBS="$(cd "$SCIPY_LIBS" && pwd)"
BLAS="$(ls "$SCIPY_LIBS"/libscipy_openblas-*.so | head -1)"
mkdir -p "$OUT"
g++ -std=c++20 -O3 -ffp-contract=off -fPIC -shared -pthread \
  -I"$REF/include" -I"$HERE/eigen_shim" \
  "$REF"/src/geometry.cpp "$REF"/src/chebyshev.cpp "$REF"/src/m2l.cpp "$REF"/src/direct.cpp \
  "$REF"/src/taskflow.cpp "$REF"/src/runtime.cpp "$REF"/src/bench.cpp \
  "$HERE/ref_driver.cpp" \
  "$BLAS" -Wl,-rpath,"$SCIPY_LIBS" \
  -o "$OUT/libtaskfmm_ref.so.tmp"
mv "$OUT/libtaskfmm_ref.so.tmp" "$OUT/libtaskfmm_ref.so"
echo "built $OUT/libtaskfmm_ref.so"
