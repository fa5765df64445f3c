#!/usr/bin/env bash
# Compile the reference implementation where it lies (/root/reference,
# read-only; nothing is copied into this repo) against the repo-owned
# Eigen-subset shim, producing oracle/_ref/znn_ref (git-ignored, but it
# travels to the GPU box with the gpurun snapshot). Used only as the parity
# pin of oracle/ and as the CPU baseline. Skipped when /root/reference is
# absent (the GPU box uses the prebuilt binary).
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF=/root/reference/proj
OUT="$HERE/../_ref"
if [ ! -d "$REF/include/znn" ]; then
    echo "reference not present; skipping oracle/_ref build"
    exit 0
fi
mkdir -p "$OUT"
SRC="$HERE/znn_ref.cpp"
BIN="$OUT/znn_ref"
if [ -x "$BIN" ] && [ "$BIN" -nt "$SRC" ] && [ "$BIN" -nt "$HERE/shim/Eigen/Core" ] && \
   [ "$BIN" -nt "$HERE/shim/unsupported/Eigen/FFT" ]; then
    exit 0
fi
# -march=x86-64-v3 (AVX2/FMA) runs on both this container and the GPU box host
g++ -std=c++20 -O3 -march=x86-64-v3 -DNDEBUG -pthread \
    -I"$HERE/shim" -I"$REF/include" -I"$REF/tests" \
    "$SRC" -o "$BIN"
echo "built $BIN"
