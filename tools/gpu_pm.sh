#!/usr/bin/env bash
# phase-major groups: parity tests, full-size c5 loss with and without, bench
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_fft.py tests/test_gpu_net.py tests/test_gpu_runtime.py tests/test_gpu_ops.py > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
tail -15 gpurun_out/pytest_quick.log
E=direct,fft,fft,fft,fft,simt
timeout 300 python tools/_net_steps.py c5 $E 3 > gpurun_out/c5_pm1.log 2>&1
ZNN_PHASE_MAJOR=0 timeout 300 python tools/_net_steps.py c5 $E 3 > gpurun_out/c5_pm0.log 2>&1
tail -n 4 gpurun_out/c5_pm1.log gpurun_out/c5_pm0.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python tools/_bench_brief.py gpurun_out/bench.log 24
