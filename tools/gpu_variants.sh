#!/usr/bin/env bash
# c5 bench under several env settings: tools/gpu_variants.sh "ENV1=a ENV2=b" "ENV1=c" ...
set -u
mkdir -p gpurun_out
i=0
for v in "$@"; do
  i=$((i+1))
  env $v timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/var_$i.log 2>&1
  echo "== [$v] rc=$?" >> gpurun_out/variants.txt
  python - gpurun_out/var_$i.log >> gpurun_out/variants.txt <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith('{')]
if not l:
    print("no result"); sys.exit()
d = json.loads(l[-1])
print("step %.2f ms" % d["ms_per_step"])
for k in d["kernel_shares"]:
    if k["ms_per_step"] > 0.7:
        print("  %7.2f %s" % (k["ms_per_step"], k["kernel"]))
PY
done
cat gpurun_out/variants.txt
