"""DRAM traffic per pass from an `ncu --set full` raw CSV of one FFT layer
(tools/gpu_ncu_transforms.sh): python tools/_traffic_json.py raw.csv out.json label::kernelA+kernelB[@occurrence] ...
Each label is a bench.py kernel_shares label; its traffic is the sum of
dram__bytes_read.sum + dram__bytes_write.sum over the named kernels' n-th launches."""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, u = rows[0], rows[1]
ik = h.index("Kernel Name")
ir, iw, it = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"), h.index("gpu__time_duration.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
launches = {}
for r in rows[2:]:
    launches.setdefault(r[ik], []).append(
        (float(r[ir]) * scale[u[ir]] + float(r[iw]) * scale[u[iw]], float(r[it]), u[it]))
out = {"source": sys.argv[1], "per_kernel": {}}
for spec in sys.argv[3:]:
    label, ks = spec.split("::", 1)
    occ = 0
    if "@" in ks:
        ks, o = ks.rsplit("@", 1)
        occ = int(o)
    tot, parts = 0.0, []
    for k in ks.split("+"):
        name = next(n for n in launches if k in n)
        b, t, tu = launches[name][occ]
        tot += b
        parts.append({"kernel": name[:80], "dram_bytes": b, "duration": t, "duration_unit": tu})
    out["per_kernel"][label] = {"dram_bytes": tot, "kernels": parts}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1)[:1500])
