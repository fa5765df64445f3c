#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
for ni in 2 1; do
ZNN_FFT_GRP_NI=$ni timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --layer-engines direct,fft,fft,fft,fft,simt > gpurun_out/bench_ni$ni.log 2>&1
echo "NI=$ni"; python tools/_bench_brief.py gpurun_out/bench_ni$ni.log 48 | grep -E "ms/step|P=20|P=16|P=12" | grep -E "ms/step|image|grad_fwd|dgrad_inv"
done
