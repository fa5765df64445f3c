#!/usr/bin/env bash
# executor-level parity (nets, runtime, FFT nets, full size) then the c5 bench
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_net.py tests/test_gpu_runtime.py tests/test_gpu_fft.py tests/test_gpu_fullsize.py tests/test_gpu_cpp_engine.py > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
tail -5 gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python tools/_bench_brief.py gpurun_out/bench.log ${1:-12}
