#!/usr/bin/env bash
# numbers for DESIGN sections 7 / 8: per-rank steps at the local batches of 1-8 ranks, the other configs
set -u
mkdir -p gpurun_out
timeout 1200 python tools/_rank_batches.py c5 16 8 4 2 > gpurun_out/rank_batches_c5.log 2>&1
tail -8 gpurun_out/rank_batches_c5.log
for c in c1 c2 c3 c4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
  python tools/_bench_brief.py gpurun_out/bench_$c.log 0 | head -1
done
