#!/bin/sh
# Builds oracle/_ref/libfskin_ref.so from the REFERENCE'S OWN hot-path sources where they lie under
# /root/reference (never copied into this repo), with the reference's own flags (proj/CMakeLists.txt:
# C++20 with CMake's default GNU extensions, Release -O3; -march=native pinned to x86-64-v3 — AVX2 + FMA,
# the same contraction as any FMA host without depending on this container's AVX-512), against oracle/eigen_shim
# (the Eigen3 stand-in; Eigen3 is absent from this image). Test infrastructure only. No-op without
# /root/reference (the GPU box uses the prebuilt .so that travels with the snapshot).
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
REF=${FSK_REFERENCE:-/root/reference/proj}
[ -d "$REF/src" ] || { echo "ref_build: $REF not found, skipped"; exit 0; }
mkdir -p "$HERE/_ref"
${CXX:-g++} -std=gnu++20 -O3 -march=x86-64-v3 -DNDEBUG -fPIC -shared -pthread -w \
    -I "$HERE/eigen_shim" -I "$REF/include" \
    "$REF/src/geometry.cpp" "$REF/src/skinning.cpp" "$REF/src/deformer.cpp" "$REF/src/correspondence.cpp" \
    "$HERE/ref_stubs.cpp" "$HERE/ref_capi.cpp" -o "$HERE/_ref/libfskin_ref.so"
echo "ref_build: $HERE/_ref/libfskin_ref.so"
