#!/usr/bin/env bash
# Round-2 evidence pass: smoke, GPU suite, c5 bench (with the reference CPU
# baseline), ncu launch list of one bench step with the autotuned engines
# fixed, c4 autotune log.  Logs under gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
ENG=direct,fft,fft,fft,fft,simt
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --layer-engines $ENG > gpurun_out/bench_fixed.log 2>&1; echo "rc=$?" >> gpurun_out/bench_fixed.log
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 950 --csv \
  --log-file gpurun_out/launches_c5_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --layer-engines $ENG > gpurun_out/ncu_launches.log 2>&1
python tools/_launch_shares.py gpurun_out/launches_c5_bench.csv > gpurun_out/launch_shares_c5_bench.txt 2>&1
timeout 600 python tools/_net_steps.py c4 auto 3 > gpurun_out/c4_autotune.log 2>&1
tail -3 gpurun_out/smoke.log; tail -4 gpurun_out/pytest_gpu.log; tail -c 300 gpurun_out/bench.log; head -30 gpurun_out/launch_shares_c5_bench.txt; tail -12 gpurun_out/c4_autotune.log
