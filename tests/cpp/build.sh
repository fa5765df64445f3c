#!/usr/bin/env bash
# Build the reference-side drop-in test (tests/cpp/gpu_engine_round.cpp):
# include/znn_gpu_engine.hpp compiled against the reference's headers where
# they lie (/root/reference/proj, read-only; nothing copied) with the repo's
# Eigen-subset shim, linked with paper_1510_06706_b200/libznn_cuda.so.
# Output: oracle/_ref/gpu_engine_round (git-ignored, travels to the GPU box).
# Skipped when /root/reference is absent (the GPU box uses the prebuilt file).
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
ROOT="$(cd "$HERE/../.." && pwd)"
REF=/root/reference/proj
OUT="$ROOT/oracle/_ref"
if [ ! -d "$REF/include/znn" ]; then
    echo "reference not present; skipping gpu_engine_round build"
    exit 0
fi
mkdir -p "$OUT"
BIN="$OUT/gpu_engine_round"
SRC="$HERE/gpu_engine_round.cpp"
HDR="$ROOT/include/znn_gpu_engine.hpp"
if [ -x "$BIN" ] && [ "$BIN" -nt "$SRC" ] && [ "$BIN" -nt "$HDR" ] && [ "$BIN" -nt "$ROOT/include/znn_cuda.h" ]; then
    exit 0
fi
g++ -std=c++20 -O2 -march=x86-64-v3 -pthread \
    -I"$ROOT/include" -I"$ROOT/oracle/ref/shim" -I"$REF/include" -I"$REF/tests" \
    "$SRC" -o "$BIN" -L"$ROOT/paper_1510_06706_b200" -lznn_cuda \
    -Wl,-rpath,'$ORIGIN/../../paper_1510_06706_b200'
echo "built $BIN"
