#!/usr/bin/env bash
# ncu --set full of kernels (regex, first N launches) inside one c5 bench step (engines fixed)
#   tools/gpu_ncu_bench.sh <regex> <count> <tag>
set -u
mkdir -p gpurun_out /tmp/ncu
R=$1; N=$2; T=$3
E=direct,fft,fft,fft,fft,simt
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --layer-engines $E > gpurun_out/ncu_bench_plain.log 2>&1 || exit 1
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name regex:"$R" --launch-count $N \
  -o /tmp/ncu/$T -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --layer-engines $E > gpurun_out/ncu_$T.log 2>&1
ncu -i /tmp/ncu/$T.ncu-rep --page raw --csv > gpurun_out/ncu_${T}_raw.csv 2>/dev/null
ncu -i /tmp/ncu/$T.ncu-rep --page source --csv > gpurun_out/ncu_${T}_source.csv 2>/dev/null
