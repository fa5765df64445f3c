"""Per-layer gradient comparison FFT vs direct engine (debug helper, not a
test): python tools/_fft_grad_check.py [config] [width_div]"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1510_06706_b200 import Context, Net, configs as C  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else 'c4'
wd = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cfg = C.scaled(name, wd, (2, 2, 2) if name != 'c2' else (1, 6, 6), batch=2)
ctx = Context(0)
rng = np.random.default_rng(5)
params = C.init_params(cfg, 5)
x = rng.uniform(0, 1, size=(cfg.batch, cfg.in_maps) + tuple(cfg.in_dims)).astype(np.float32)
lab = (rng.uniform(size=(cfg.batch, cfg.layers[-1].width) + tuple(cfg.out_dims)) < 0.5).astype(np.float32)
import os
nconv = len(cfg.conv_layers())
res = {}
for mode in ('direct', 'fft', 'fft_dense'):
    if mode == 'fft_dense':
        os.environ['ZNN_FFT_DENSE_KERNELS'] = '1'
    net = Net(ctx, cfg.netspec(), cfg.out_dims, batch=cfg.batch, lr=cfg.lr, momentum=cfg.momentum, loss=cfg.loss)
    if mode != 'direct':
        for li in range(nconv - 1):
            net.set_layer_engine(li, 'fft')
    net.set_params(params)
    xs = torch.as_tensor(x, device='cuda')
    ls = torch.as_tensor(lab, device='cuda')
    loss = net.forward_backward(xs, ls)
    res[mode] = (loss, net.get_gradients().copy())
gd = res['direct'][1]
for mode in ('fft', 'fft_dense'):
    gf = res[mode][1]
    d = np.abs(gd - gf)
    print(mode, 'loss', res['direct'][0], res[mode][0], 'max|g|', np.abs(gd).max(), 'max diff', d.max(),
          'n bad', int((d > 1e-3 * np.abs(gd).max()).sum()), 'of', gd.size)
    idx = np.argsort(-d)[:8]
    print('  worst idx', idx.tolist(), 'direct', gd[idx].round(6).tolist(), mode, gf[idx].round(6).tolist())
