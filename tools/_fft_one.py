"""One FFT-engine step of c4 scaled (debug helper for compute-sanitizer)."""
import sys
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
gs = []
for rep in range(2):
    net = Net(ctx, cfg.netspec(), cfg.out_dims, batch=2, lr=cfg.lr, momentum=cfg.momentum, loss="ce")
    for li in range(3):
        net.set_layer_engine(li, "fft")
    net.set_params(params)
    net.forward_backward(xs, ls)
    gs.append(net.get_gradients().copy())
print('rep diff', np.abs(gs[0] - gs[1]).max(), 'at', int(np.abs(gs[0] - gs[1]).argmax()))

# mask / activation comparison against the direct engine
res = {}
for mode in ("direct", "fft"):
    net = Net(ctx, cfg.netspec(), cfg.out_dims, batch=2, lr=cfg.lr, momentum=cfg.momentum, loss="ce")
    if mode == "fft":
        for li in range(3):
            net.set_layer_engine(li, "fft")
    net.set_params(params)
    net.forward_backward(xs, ls)
    acts, masks = [], []
    gi = 0
    while True:
        try:
            info = net.group_info(gi)
        except Exception:
            break
        try:
            acts.append(net.group_image(gi, 0))
        except Exception:
            acts.append(None)
            gi += 1
            masks.append(None)
            continue
        try:
            masks.append(net.group_mask(gi))
        except Exception:
            masks.append(None)
        gi += 1
    res[mode] = (acts, masks)
for gi, (a, b) in enumerate(zip(res["direct"][0], res["fft"][0])):
    if a is None:
        continue
    ma, mb = res["direct"][1][gi], res["fft"][1][gi]
    md = None if ma is None else int((ma != mb).sum())
    print('group', gi, 'act max diff', float(np.abs(a - b).max()), 'rel', float(np.abs(a - b).max() / (np.abs(a).max() + 1e-30)), 'mask mismatches', md)
