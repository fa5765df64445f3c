#!/usr/bin/env bash
# quick GPU pass: selected pytest files (args) then a short c5 bench
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu "$@" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
tail -30 gpurun_out/pytest_quick.log
if grep -q "pytest rc=0" gpurun_out/pytest_quick.log; then
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
  tail -c 600 gpurun_out/bench.log
fi
