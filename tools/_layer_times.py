"""Per-layer, per-pass device timings of one config's conv layers (profiling
helper, not a test): python tools/_layer_times.py c5 [engine ...]"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1510_06706_b200 import Context, configs as C, ops  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else 'c5'
engines = sys.argv[2:] or ['direct']
cfg = C.CONFIGS[name]
B = cfg.batch
ctx = Context(0)
st = torch.cuda.current_stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    b.synchronize()
    return a.elapsed_time(b) / reps


tot = {}
for li, (kind, fi, fo, n, m, k, s) in enumerate(C.layer_shapes(cfg)):
    if kind != 'conv':
        continue
    x = torch.rand((B, fi) + tuple(n), device='cuda')
    w = (torch.rand((fo, fi) + tuple(k), device='cuda') - 0.5) * 0.02
    g = torch.rand((B, fo) + tuple(m), device='cuda') - 0.5
    fl = 2.0 * B * fi * fo * np.prod(m) * np.prod(k)
    for eng in engines:
        tf = timed(lambda: ops.conv_fwd(ctx, x, w, k, s, act='relu', engine=eng))
        td = timed(lambda: ops.conv_dgrad(ctx, g, w, k, s, engine=eng)) if li > 0 and fi > 1 else 0.0
        tw = timed(lambda: ops.conv_wgrad(ctx, x, g, k, s, engine=eng))
        tot[eng] = tot.get(eng, 0.0) + tf + td + tw
        print(f'{eng:6s} L{li} {fi:4d}->{fo:4d} n={tuple(n)} k={tuple(k)} s={tuple(s)}: '
              f'fwd {tf:8.2f} ms {fl / tf / 1e9 if tf else 0:6.1f} | dgrad {td:8.2f} ms '
              f'{fl / td / 1e9 if td else 0:6.1f} | wgrad {tw:8.2f} ms {fl / tw / 1e9 if tw else 0:6.1f} TFLOP/s',
              flush=True)
    del x, w, g
    torch.cuda.empty_cache()
for eng, t in tot.items():
    print(f'{eng}: conv total {t:.1f} ms', flush=True)
