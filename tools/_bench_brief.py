"""Brief view of a bench.py JSON line: python tools/_bench_brief.py gpurun_out/bench.log [n]"""
import json
import sys

l = [x for x in open(sys.argv[1]) if x.startswith('{')][-1]
d = json.loads(l)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 48
print("ms/step %.2f  value %.4g  e2e %.4g  graph %.2f  launches %d  engines %s" % (
    d['ms_per_step'], d['value'], d['e2e']['value'], d.get('graph_ms_per_step') or 0, d['gpu_launches'],
    d['config'].get('conv_engines')))
r = d['roofline']
print("roofline: %s frac %.3f (%.0f GB/s)" % (r['kernel'], r['frac'], r['achieved']))
for k in d['kernel_shares'][:n]:
    print("%7.3f ms %5.1f%% %7.0f GB/s  %s" % (k['ms_per_step'], 100 * k['share_of_step'], k['gbs'], k['kernel']))
