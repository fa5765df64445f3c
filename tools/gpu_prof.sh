#!/usr/bin/env bash
# ncu captures of the FFT engine's top kernels at c5 conv2 / conv3 (after the
# program ran clean without ncu); raw-page CSVs under gpurun_out/ (the .ncu-rep
# files stay on the box: gpurun copies back at most 64 MiB)
set -u
mkdir -p gpurun_out /tmp/ncu
timeout 300 python tools/prof_layer.py c5 1 1 > gpurun_out/prof_layer.log 2>&1 || exit 1
for spec in "cmac_ss_k 1" "cmac_upd_ss_k 1" "fft3_fwd_small_k 2" "fft3_inv_small_k 2"; do
  set -- $spec
  K=$1; LI=$2
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:$K --launch-count 1 \
    -o /tmp/ncu/$K -f python tools/prof_layer.py c5 $LI 1 > gpurun_out/ncu_$K.log 2>&1
  ncu -i /tmp/ncu/$K.ncu-rep --page raw --csv > gpurun_out/ncu_${K}_raw.csv 2>/dev/null
  ncu -i /tmp/ncu/$K.ncu-rep --page details --csv > gpurun_out/ncu_${K}_details.csv 2>/dev/null
done
ls -la gpurun_out/
