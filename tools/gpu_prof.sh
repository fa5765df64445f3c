#!/usr/bin/env bash
# ncu captures of the FFT engine's top kernels at c5 conv2 (after the program
# ran clean without ncu); outputs under gpurun_out/
set -u
mkdir -p gpurun_out
timeout 300 python tools/prof_layer.py c5 1 1 > gpurun_out/prof_layer.log 2>&1 || exit 1
for K in cmac_ss_k cmac_upd_ss_k fft3_fwd_small_k fft3_inv_small_k; do
  L=1; [ "$K" = "fft3_fwd_small_k" ] || [ "$K" = "fft3_inv_small_k" ] && L=2
  LI=1; [ "$K" = "fft3_fwd_small_k" ] || [ "$K" = "fft3_inv_small_k" ] && LI=2
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:$K --launch-count 1 \
    -o gpurun_out/ncu_$K -f python tools/prof_layer.py c5 $LI 1 > gpurun_out/ncu_$K.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
