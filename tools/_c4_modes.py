"""Time a c4 step per engine assignment (profiling helper)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1510_06706_b200 import Context, Net, configs as C
cfg = C.CONFIGS['c4']
ctx = Context(0)
rng = np.random.default_rng(0)
x = torch.as_tensor(rng.uniform(0, 1, size=(8, 1) + cfg.in_dims).astype(np.float32), device='cuda')
lab = torch.as_tensor((rng.uniform(size=(8, 3) + cfg.out_dims) < 0.5).astype(np.float32), device='cuda')
modes = {'direct': ['direct'] * 4, 'fft': ['fft', 'fft', 'fft', 'direct'], 'fft23': ['direct', 'fft', 'fft', 'direct']}
only = sys.argv[1:] or list(modes)
for name in only:
    net = Net(ctx, cfg.netspec(), cfg.out_dims, batch=8, lr=0.01, momentum=0.9, loss='ce')
    for i, e in enumerate(modes[name]):
        net.set_layer_engine(i, e)
    net.set_params(C.init_params(cfg, 1))
    for _ in range(2):
        net.forward_backward(x, lab, sync_loss=False); net.apply_update()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(3):
        net.forward_backward(x, lab, sync_loss=False); net.apply_update()
    torch.cuda.synchronize()
    print(name, f'{(time.perf_counter() - t0) / 3 * 1e3:.2f} ms/step', flush=True)
    del net
