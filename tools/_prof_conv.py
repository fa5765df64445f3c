"""One fwd / dgrad / wgrad launch of a conv layer shape, for ncu captures
(profiling helper, not a test): python tools/_prof_conv.py B fi fo n k s"""
import sys

import torch

sys.path.insert(0, '.')
from paper_1510_06706_b200 import Context, ops  # noqa: E402

B, fi, fo, n, k, s = (int(a) for a in (sys.argv[1:7] if len(sys.argv) >= 7 else (1, 120, 120, 80, 5, 4)))
passes = sys.argv[7].split(',') if len(sys.argv) > 7 else ['fwd', 'dgrad', 'wgrad']
ctx = Context(0)
n3, k3, s3 = (n, n, n), (k, k, k), (s, s, s)
m = n - s * (k - 1)
x = torch.rand((B, fi) + n3, device='cuda')
w = (torch.rand((fo, fi) + k3, device='cuda') - 0.5) * 0.02
g = torch.rand((B, fo, m, m, m), device='cuda') - 0.5
for p in passes:
    if p == 'fwd':
        ops.conv_fwd(ctx, x, w, k3, s3, act='relu')
    elif p == 'dgrad':
        ops.conv_dgrad(ctx, g, w, k3, s3)
    else:
        ops.conv_wgrad(ctx, x, g, k3, s3)
torch.cuda.synchronize()
print('ok', flush=True)
