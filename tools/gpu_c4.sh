#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_fft.py > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
tail -4 gpurun_out/pytest_quick.log
timeout 600 python tools/_net_steps.py c4 auto 3 > gpurun_out/c4_autotune.log 2>&1
tail -9 gpurun_out/c4_autotune.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python tools/_bench_brief.py gpurun_out/bench.log 6
