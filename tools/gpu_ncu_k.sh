#!/usr/bin/env bash
# ncu --set full of one kernel (regex) of one FFT layer at full shape:
#   tools/gpu_ncu_k.sh <config> <conv layer> <kernel regex> [tag]
set -u
mkdir -p gpurun_out /tmp/ncu
C=$1; L=$2; K=$3; T=${4:-$K}
timeout 300 python tools/prof_layer.py $C $L 1 > gpurun_out/prof_layer_$C$L.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"$K" --launch-count 1 \
  -o /tmp/ncu/$T -f python tools/prof_layer.py $C $L 1 > gpurun_out/ncu_$T.log 2>&1
ncu -i /tmp/ncu/$T.ncu-rep --page raw --csv > gpurun_out/ncu_${T}_raw.csv 2>/dev/null
ncu -i /tmp/ncu/$T.ncu-rep --page source --csv > gpurun_out/ncu_${T}_source.csv 2>/dev/null
ncu -i /tmp/ncu/$T.ncu-rep --page details --csv > gpurun_out/ncu_${T}_details.csv 2>/dev/null
