#!/usr/bin/env bash
# One gpurun pass: smoke, the GPU suite (optionally a -k filter), a short bench.
# usage: tools/gpu_check.sh [pytest -k expr] ; logs under gpurun_out/
set -u
mkdir -p gpurun_out
K="${1:-}"
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests -x -q -m gpu -k "$K" > gpurun_out/pytest_gpu.log 2>&1
else
  timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -3 gpurun_out/smoke.log gpurun_out/pytest_gpu.log; tail -c 1500 gpurun_out/bench.log
