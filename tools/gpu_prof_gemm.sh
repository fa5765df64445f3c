#!/usr/bin/env bash
# ncu --set full of the tensor-core CMAC GEMM (and its operand transposes) at
# c5 conv2 (layer 1) and conv3 (layer 2); raw / source CSVs under gpurun_out/
set -u
mkdir -p gpurun_out /tmp/ncu
for LI in 1 2; do
  timeout 300 python tools/prof_layer.py c5 $LI 1 > gpurun_out/prof_layer_$LI.log 2>&1 || exit 1
done
for LI in 1 2; do
  for K in ${KERNELS:-cgemm_tc_k}; do
    timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:$K --launch-count 1 \
      -o /tmp/ncu/${K}_$LI -f python tools/prof_layer.py c5 $LI 1 > gpurun_out/ncu_${K}_$LI.log 2>&1
    ncu -i /tmp/ncu/${K}_$LI.ncu-rep --page raw --csv > gpurun_out/ncu_${K}_${LI}_raw.csv 2>/dev/null
    ncu -i /tmp/ncu/${K}_$LI.ncu-rep --page details --csv > gpurun_out/ncu_${K}_${LI}_details.csv 2>/dev/null
    ncu -i /tmp/ncu/${K}_$LI.ncu-rep --page source --csv > gpurun_out/ncu_${K}_${LI}_source.csv 2>/dev/null
  done
done
ls -la gpurun_out/
