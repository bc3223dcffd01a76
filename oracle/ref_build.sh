#!/usr/bin/env bash
# Compiles the UNMODIFIED reference headers (where they lie under /root/reference) against the clean-room
# Eigen shim into oracle/_ref/libsplat_ref.so. TEST INFRASTRUCTURE. No reference source is copied.
# The reference's own build system is not used (its CMakeLists.txt has no targets and expects a vendored
# Eigen that is absent); this is the whole recipe.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF="${SPLAT_REFERENCE:-/root/reference}/proj/include"
[ -f "$REF/splat/projection.hpp" ] || { echo "reference headers not found under $REF" >&2; exit 3; }
mkdir -p "$HERE/_ref"
# -ffp-contract=off: no FMA contraction, so results are the plain IEEE evaluation of the reference's expressions
g++ -std=c++20 -O2 -fPIC -shared -ffp-contract=off -Wall -Wno-unused-parameter \
    -I"$HERE/eigen_shim" -I"$REF" "$HERE/ref_harness.cpp" -o "$HERE/_ref/libsplat_ref.so.tmp" -pthread
mv "$HERE/_ref/libsplat_ref.so.tmp" "$HERE/_ref/libsplat_ref.so"
echo "built $HERE/_ref/libsplat_ref.so"
