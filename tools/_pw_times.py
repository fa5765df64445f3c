"""Device time and achieved HBM GB/s of the pointwise / max-filter passes at
c5 sizes (profiling helper, not a test): python tools/_pw_times.py [B]"""
import sys

import torch

sys.path.insert(0, '.')
from paper_1510_06706_b200 import Context, ops  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
ctx = Context(0)
st = torch.cuda.current_stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    b.synchronize()
    return a.elapsed_time(b) / reps


f = 120
for (n, k, s) in [((91, 91, 91), (2, 2, 2), (1, 1, 1)), ((82, 82, 82), (2, 2, 2), (2, 2, 2))]:
    x = torch.rand((B, f) + n, device='cuda')
    y, mask = ops.maxfilter_fwd(ctx, x, k, s)
    m = y.shape[2:]
    g = torch.rand_like(y)
    nin, nout = x.numel(), y.numel()
    tf = timed(lambda: ops.maxfilter_fwd(ctx, x, k, s))
    tb = timed(lambda: ops.maxfilter_bwd(ctx, g, mask, k, s))
    bf = 4 * nin + 8 * nout
    bb = 8 * nout + 4 * nin
    print(f'maxfilter n={n} s={s}: fwd {tf:.2f} ms {bf / tf / 1e6:.0f} GB/s | bwd {tb:.2f} ms {bb / tb / 1e6:.0f} GB/s',
          flush=True)
    del x, y, mask, g
    torch.cuda.empty_cache()
n = (90, 90, 90)
g = torch.rand((B, f) + n, device='cuda')
yv = torch.rand_like(g)
t = timed(lambda: ops.transfer_bwd(ctx, g, yv, ['relu'] * f, from_output=True))
print(f'transfer_bwd n={n}: {t:.2f} ms {12 * g.numel() / t / 1e6:.0f} GB/s', flush=True)
