#!/usr/bin/env bash
# ncu --set full of the FFT transforms at c5 conv2 (P = 48: z + xy register
# passes) and conv3 (P = 20: fused cube kernels), one layer fwd + bwd each
set -u
mkdir -p gpurun_out /tmp/ncu
timeout 300 python tools/prof_layer.py c5 1 1 > gpurun_out/prof_layer_c51.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on \
  --kernel-name regex:'fft_z_fwd_reg_k|fft_xy_fwd_pair_k|fft_xy_inv_pair_k|fft_z_inv_reg_k' --launch-count 8 \
  -o /tmp/ncu/tr48 -f python tools/prof_layer.py c5 1 1 > gpurun_out/ncu_tr48.log 2>&1
ncu -i /tmp/ncu/tr48.ncu-rep --page raw --csv > gpurun_out/ncu_tr48_raw.csv 2>/dev/null
ncu -i /tmp/ncu/tr48.ncu-rep --page details --csv > gpurun_out/ncu_tr48_details.csv 2>/dev/null
ncu -i /tmp/ncu/tr48.ncu-rep --page source --csv > gpurun_out/ncu_tr48_source.csv 2>/dev/null
timeout 1200 ncu --set full --clock-control none --import-source on \
  --kernel-name regex:'fft3_fwd_reg_k|fft3_inv_reg_k' --launch-count 4 \
  -o /tmp/ncu/tr20 -f python tools/prof_layer.py c5 2 1 > gpurun_out/ncu_tr20.log 2>&1
ncu -i /tmp/ncu/tr20.ncu-rep --page raw --csv > gpurun_out/ncu_tr20_raw.csv 2>/dev/null
ncu -i /tmp/ncu/tr20.ncu-rep --page details --csv > gpurun_out/ncu_tr20_details.csv 2>/dev/null
ncu -i /tmp/ncu/tr20.ncu-rep --page source --csv > gpurun_out/ncu_tr20_source.csv 2>/dev/null
ls -la gpurun_out/
