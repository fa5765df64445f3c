"""Run one FFT-engine conv layer (fwd + bwd) at a config's full shape, for
ncu captures of single kernels:  python tools/prof_layer.py c5 1  (conv
layer index among the configs' conv layers)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_06706_b200 import Context, FftPlan, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
li = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = configs.CONFIGS[name]
convs = [s for s in configs.layer_shapes(cfg) if s[0] == "conv"]
_, fi, fo, n, m, k, s = convs[li]
B = cfg.batch
ctx = Context(0)
x = torch.rand((B, fi) + tuple(n), device="cuda")
w = torch.rand((fo, fi) + tuple(k), device="cuda") * 0.01
g = torch.rand((B, fo) + tuple(m), device="cuda")
p = FftPlan(ctx, B, fi, fo, n, k, s)
for _ in range(reps):
    y = p.forward(x, w, act="relu")
    dx, dw = p.backward(g, w, want_dx=fi > 1)
torch.cuda.synchronize()
print("ok", name, li, p.info())
