"""FFT sparse-tap vs dense kernel transforms over several SGD steps (debug
helper, not a test)."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1510_06706_b200 import Context, Net, configs as C
cfg = C.scaled("c4", 16, (2, 2, 2), batch=2)
ctx = Context(0)
rng = np.random.default_rng(9)
params = C.init_params(cfg, 9)
x = rng.uniform(0, 1, size=(2, 1) + tuple(cfg.in_dims)).astype(np.float32)
lab = (rng.uniform(size=(2, 3) + tuple(cfg.out_dims)) < 0.5).astype(np.float32)
xs = torch.as_tensor(x, device='cuda'); ls = torch.as_tensor(lab, device='cuda')
nets = {}
for mode in ("fft", "fft_dense", "direct"):
    net = Net(ctx, cfg.netspec(), cfg.out_dims, batch=2, lr=cfg.lr, momentum=cfg.momentum, loss="ce")
    if mode != "direct":
        for li in range(3):
            net.set_layer_engine(li, "fft")
    net.set_params(params)
    nets[mode] = net
for step in range(3):
    r = {}
    for mode, net in nets.items():
        if mode == "fft_dense": os.environ['ZNN_FFT_DENSE_KERNELS'] = '1'
        else: os.environ.pop('ZNN_FFT_DENSE_KERNELS', None)
        loss = net.forward_backward(xs, ls)
        g = net.get_gradients().copy()
        net.apply_update()
        r[mode] = (loss, g, net.get_params().copy())
    for mode in ("fft", "fft_dense"):
        d = np.abs(r[mode][1] - r["direct"][1]); p = np.abs(r[mode][2] - r["direct"][2])
        print(step, mode, 'loss', r[mode][0], r["direct"][0], 'grad diff', d.max(), 'argmax', int(d.argmax()), 'param diff', p.max())
