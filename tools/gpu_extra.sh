set -u
mkdir -p gpurun_out
timeout 900 python tools/_rank_batches.py c5 16 8 4 2 > gpurun_out/rank_batches_c5.log 2>&1
for c in c4 c3 c2 c1; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
done
timeout 1200 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref_c5.log 2>&1
nproc > gpurun_out/nproc.txt; lscpu >> gpurun_out/nproc.txt 2>&1; free -g >> gpurun_out/nproc.txt
