"""One launch each of the tc conv fwd / dgrad / wgrad at a c5 layer shape (profiling helper)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1510_06706_b200 import Context, ops
ctx = Context(0)
B, fi, fo, n, k, s = 1, 120, 120, (80, 80, 80), (5, 5, 5), (4, 4, 4)
if len(sys.argv) > 1 and sys.argv[1] == 'c5conv2':
    B, fi, fo, n, k, s = 1, 120, 120, (90, 90, 90), (5, 5, 5), (2, 2, 2)
x = torch.rand((B, fi) + n, device='cuda'); w = (torch.rand((fo, fi) + k, device='cuda') - 0.5) * 0.01
m = [n[a] - s[a] * (k[a] - 1) for a in range(3)]
g = torch.rand((B, fo) + tuple(m), device='cuda') - 0.5
for _ in range(2):
    ops.conv_fwd(ctx, x, w, k, s, act='relu')
    ops.conv_dgrad(ctx, g, w, k, s)
    ops.conv_wgrad(ctx, x, g, k, s)
torch.cuda.synchronize()
print('ok')
