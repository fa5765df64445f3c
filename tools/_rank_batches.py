"""Per-rank step time of a config at the local batch each of N data-parallel
ranks would hold (B/N), autotuned per batch (profiling helper, not a test):
python tools/_rank_batches.py c5 16 8 4 2 1"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1510_06706_b200 import Context, Net, configs as C  # noqa: E402
from paper_1510_06706_b200.api import profile_enable, profile_report  # noqa: E402

name = sys.argv[1]
batches = [int(v) for v in sys.argv[2:] if not v.startswith('--')]
ctx = Context(0)
for Bl in batches:
    cfg = C.CONFIGS[name]
    rng = np.random.default_rng(0)
    x = torch.as_tensor(rng.uniform(0, 1, size=(Bl, cfg.in_maps) + cfg.in_dims).astype(np.float32), device='cuda')
    lab = torch.as_tensor((rng.uniform(size=(Bl, cfg.layers[-1].width) + cfg.out_dims) < 0.5).astype(np.float32),
                          device='cuda')
    net = Net(ctx, cfg.netspec(), cfg.out_dims, batch=Bl, global_batch=cfg.batch, lr=cfg.lr, momentum=cfg.momentum,
              loss=cfg.loss, engine="auto")
    net.set_params(C.init_params(cfg, 1))
    for _ in range(2):
        net.train_step(x, lab, sync_loss=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        net.train_step(x, lab, sync_loss=False)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 3
    N = cfg.batch // Bl
    print(f'{name} local batch {Bl:2d} (N = {N}): {ms:8.2f} ms/step, engines {net.engines}, '
          f'projected {N}-GPU throughput {cfg.batch * np.prod(cfg.out_dims) / (ms * 1e-3):.3g} voxels/s', flush=True)
    if '--shares' in sys.argv:
        profile_report(ctx)
        profile_enable(ctx, True)
        net.train_step(x, lab, sync_loss=False)
        torch.cuda.synchronize()
        profile_enable(ctx, False)
        for e in sorted(profile_report(ctx), key=lambda e: -e['ms'])[:22]:
            print(f"   {e['ms']:7.3f} ms  {e['kernel']}", flush=True)
    net.close()
    del x, lab
    torch.cuda.empty_cache()
