"""Wall-clock timing of the c5 conv1 forward (1 -> 120, 95^3, 5^3, B = 16) on
the direct engine (profiling helper): python tools/_conv1_time.py"""
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_1510_06706_b200 import Context, ops  # noqa: E402

ctx = Context(0)
x = torch.rand((16, 1, 95, 95, 95), device="cuda")
w = torch.rand((120, 1, 5, 5, 5), device="cuda") * 0.1
b = torch.rand(120, device="cuda")
for _ in range(2):
    y = ops.conv_fwd(ctx, x, w, (5, 5, 5), bias=b, act="relu")
torch.cuda.synchronize()
t = time.time()
for _ in range(10):
    y = ops.conv_fwd(ctx, x, w, (5, 5, 5), bias=b, act="relu")
torch.cuda.synchronize()
print("conv1 fwd %.3f ms" % ((time.time() - t) / 10 * 1e3))
