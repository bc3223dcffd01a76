#!/usr/bin/env bash
# Builds tests/cpp/_build/facade_test: a C++ caller of the reference API + the drop-in façade. Needs the reference
# headers (/root/reference) and uses oracle/eigen_shim for the Eigen the reference does not vendor.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
ROOT="$(cd "$HERE/../.." && pwd)"
REF="${SPLAT_REFERENCE:-/root/reference}/proj/include"
[ -f "$REF/splat/projection.hpp" ] || { echo "reference headers not found under $REF" >&2; exit 3; }
mkdir -p "$HERE/_build"
g++ -std=c++20 -O2 -ffp-contract=off -Wall -Wno-unused-parameter -I"$ROOT/include" -I"$ROOT/oracle/eigen_shim" -I"$REF" \
    "$HERE/facade_test.cpp" -o "$HERE/_build/facade_test" \
    -L"$ROOT/paper_2411_16816_b200" -lsplat_b200 -Wl,-rpath,'$ORIGIN/../../../paper_2411_16816_b200' \
    -Wl,-rpath,/usr/local/cuda/lib64 -L/usr/local/cuda/lib64 -lcudart -pthread
echo "built $HERE/_build/facade_test"
