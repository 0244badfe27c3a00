#!/usr/bin/env bash
# Builds the CPU restatement (oracle/restate) -> oracle/_build/liboracle.so.
# Test infrastructure only; -ffp-contract=off keeps the FP64 geometry plain IEEE.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
mkdir -p "$HERE/_build"
g++ -std=c++20 -O2 -ffp-contract=off -fPIC -shared "$HERE/restate/fmm_oracle.cpp" -o "$HERE/_build/liboracle.so.tmp"
mv "$HERE/_build/liboracle.so.tmp" "$HERE/_build/liboracle.so"
echo "built $HERE/_build/liboracle.so"
