#!/usr/bin/env bash
# full GPU pass: smoke, whole GPU suite, c5 bench (3 warm-up, 5 steps), rank-batch projection
set -u
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python tools/_rank_batches.py c5 16 8 4 2 > gpurun_out/rank_batches_c5.log 2>&1
tail -3 gpurun_out/smoke.log; tail -4 gpurun_out/pytest_gpu.log; tail -c 400 gpurun_out/bench.log; cat gpurun_out/rank_batches_c5.log | tail -6
