"""Run W+K training steps of a config with fixed per-layer engines (profiling
helper, not a test): python tools/_net_steps.py c4 fft,fft,fft,direct|auto [steps]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1510_06706_b200 import Context, Net, configs as C  # noqa: E402

name = sys.argv[1]
engines = sys.argv[2].split(',') if len(sys.argv) > 2 else None
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = C.CONFIGS[name]
ctx = Context(0)
rng = np.random.default_rng(0)
B = cfg.batch
x = torch.as_tensor(rng.uniform(0, 1, size=(B, cfg.in_maps) + cfg.in_dims).astype(np.float32), device='cuda')
nout = cfg.layers[-1].width
lab = torch.as_tensor((rng.uniform(size=(B, nout) + cfg.out_dims) < 0.5).astype(np.float32), device='cuda')
net = Net(ctx, cfg.netspec(), cfg.out_dims, batch=B, lr=cfg.lr, momentum=cfg.momentum, loss=cfg.loss)
net.set_params(C.init_params(cfg, 1))
if engines == ['auto']:
    net.forward_backward(x, lab)
    print(net.autotune(3), flush=True)
    print('\n'.join(l for l in net.describe().splitlines() if 'autotune' in l), flush=True)
elif engines:
    for i, e in enumerate(engines):
        net.set_layer_engine(i, e)
for i in range(steps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    loss = net.forward_backward(x, lab, sync_loss=(i == steps - 1))
    net.apply_update()
    torch.cuda.synchronize()
    print(f'step {i}: {(time.perf_counter() - t0) * 1e3:.2f} ms' + (f' loss {loss:.9g}' if i == steps - 1 else ''), flush=True)
print('\n'.join(l for l in net.describe().splitlines() if 'phase-major' in l), flush=True)
