"""Weight-gradient device time of c5's conv layers under environment
overrides (profiling helper, not a test):
python tools/_wg_sweep.py c5 ZNN_WGRAD_SPLITS=0,5,10,20"""
import os
import sys

import torch

sys.path.insert(0, '.')
from paper_1510_06706_b200 import Context, configs as C, ops  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else 'c5'
var, vals = sys.argv[2].split('=') if len(sys.argv) > 2 else ('ZNN_WGRAD_SPLITS', '0')
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


for li, (kind, fi, fo, n, m, k, s) in enumerate(C.layer_shapes(cfg)):
    if kind != 'conv':
        continue
    x = torch.rand((B, fi) + tuple(n), device='cuda')
    g = torch.rand((B, fo) + tuple(m), device='cuda') - 0.5
    row = []
    for v in vals.split(','):
        if v == '0':
            os.environ.pop(var, None)
        else:
            os.environ[var] = v
        row.append(f'{v}: {timed(lambda: ops.conv_wgrad(ctx, x, g, k, s)):7.2f}')
    print(f'L{li} {fi}->{fo} n={tuple(n)} s={tuple(s)} wgrad ms | ' + ' | '.join(row), flush=True)
    del x, g
    torch.cuda.empty_cache()
