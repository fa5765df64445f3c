"""Per-kernel shares of an ncu launch list (profiling helper, not a test):
python tools/_launch_shares.py launches.csv
The csv is `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv` output; times are cold-cache and serialised,
so compare shares, not absolutes."""
import csv
import re
import sys
from collections import defaultdict

rows = [l for l in open(sys.argv[1]) if not l.startswith('==')]
per = defaultdict(dict)
names = {}
for r in csv.DictReader(rows):
    v = float(r['Metric Value'].replace(',', ''))
    unit = r['Metric Unit']
    if unit in ('ns',):
        v *= 1e-6
    elif unit == 'us':
        v *= 1e-3
    elif unit == 'ms':
        pass
    elif unit.lower() in ('byte', 'kbyte', 'mbyte', 'gbyte'):
        v *= {'byte': 1, 'kbyte': 1e3, 'mbyte': 1e6, 'gbyte': 1e9}[unit.lower()]
    per[r['ID']][r['Metric Name']] = v
    names[r['ID']] = re.sub(r'\(.*', '', r['Kernel Name']).replace('void ', '')[:60]
agg = defaultdict(lambda: [0.0, 0.0, 0])
for i, m in per.items():
    a = agg[names[i]]
    a[0] += m.get('gpu__time_duration.sum', 0.0)
    a[1] += m.get('dram__bytes_read.sum', 0.0) + m.get('dram__bytes_write.sum', 0.0)
    a[2] += 1
tot = sum(a[0] for a in agg.values())
print(f'total {tot:.1f} ms over {sum(a[2] for a in agg.values())} launches')
for n, (t, b, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f'{100 * t / tot:6.2f}% {t:9.2f} ms n={c:4d} {n:60s} {b / 1e9:8.2f} GB {b / (t * 1e-3) / 1e9 if t else 0:7.0f} GB/s')
