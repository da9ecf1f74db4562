#!/bin/sh
# Builds oracle/_ref/libref_setup.so from the reference's OWN present sources
# (/root/reference/proj/src/{basis,mesh,mapping}.cpp, unmodified) against the
# Eigen-API shim in oracle/ref_build/eigen_shim.  The reference's CMake build
# is not used (it needs Eigen3, proj/CMakeLists.txt:12).  Test infrastructure
# only; skipped when /root/reference is absent (the GPU box).
set -e
REF=${REF:-/root/reference/proj}
HERE=$(cd "$(dirname "$0")" && pwd)
OUT="$HERE/../_ref"
if [ ! -d "$REF/src" ]; then
  echo "reference tree not present ($REF); skipping oracle/_ref"
  exit 0
fi
mkdir -p "$OUT"
CXX=${CXX:-g++}
[ -x /usr/bin/g++ ] && CXX=/usr/bin/g++
$CXX -std=c++20 -O2 -fPIC -shared -I"$HERE/eigen_shim" -I"$REF/include" \
  "$REF/src/basis.cpp" "$REF/src/mesh.cpp" "$REF/src/mapping.cpp" "$HERE/ref_capi.cpp" \
  -o "$OUT/libref_setup.so"
echo "built $OUT/libref_setup.so"
