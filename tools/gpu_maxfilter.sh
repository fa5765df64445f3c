#!/usr/bin/env bash
# max-filter / pointwise check: net-level parity then the per-kernel lines of a c5 bench step
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_net.py > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
tail -3 gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --layer-engines direct,fft,fft,fft,fft,simt > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python tools/_bench_brief.py gpurun_out/bench.log 48 | grep -E "ms/step|maxfilter"
