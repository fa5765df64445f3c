#!/usr/bin/env bash
# ncu launch list (per-kernel durations) of one FFT layer at full shape:
#   tools/gpu_launches.sh <config> <conv layer index>
set -u
mkdir -p gpurun_out
C=${1:-c5}; L=${2:-2}
timeout 300 python tools/prof_layer.py $C $L 1 > gpurun_out/prof_layer_$C$L.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_$C$L.csv python tools/prof_layer.py $C $L 1 > /dev/null 2>&1
python - "$C" "$L" <<'PY'
import csv, sys, collections
C, L = sys.argv[1], sys.argv[2]
lines = open(f"gpurun_out/launches_{C}{L}.csv").read().splitlines()
rows = list(csv.reader(lines[[i for i, l in enumerate(lines) if l.startswith("\"ID\"")][0]:]))
hdr = rows[0]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    if len(r) < len(hdr): continue
    k = r[ik][:60]
    d = agg.setdefault(k, collections.defaultdict(float))
    try:
        d[r[im]] += float(r[iv].replace(",", ""))
    except ValueError:
        pass
with open(f"gpurun_out/launches_{C}{L}.txt", "w") as f:
    for k, d in agg.items():
        ms = d["gpu__time_duration.sum"] / 1e6
        gb = (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) / 1e9
        f.write(f"{ms:9.3f} ms {gb:8.2f} GB {gb / max(ms, 1e-9):7.2f} TB/s  {k}\n")
PY
cat gpurun_out/launches_$C$L.txt
