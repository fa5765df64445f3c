"""Data-parallel step logic (paper_1510_06706_b200.distributed) on CPU with the
gloo backend, world size 2: each rank computes its shard's gradients (the
oracle stands in for the CUDA executor), DataParallelStep allreduces the flat
gradient buffer and applies the update; the result must equal one
full-batch step on a single process."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


class OracleNet:
    """Stand-in with the executor's DP interface (forward_backward /
    grad_tensor / apply_update): gradients pre-scaled by 1/B_global."""

    def __init__(self, g, params, global_batch, lr, mu, loss):
        self.g, self.gb, self.lr, self.mu, self.loss = g, global_batch, lr, mu, loss
        self.p = torch.tensor(params, dtype=torch.float64)
        self.v = torch.zeros_like(self.p)
        self.grad = torch.zeros_like(self.p)
        self.losses = []

    def forward_backward(self, inputs, labels, sync_loss=False):
        acc = np.zeros(self.p.numel())
        tot = 0.0
        for x, lab in zip(inputs, labels):
            l, gr, *_ = O.patch_gradients(self.g, self.p.numpy(), x, lab, self.loss)
            acc += gr
            tot += l
        self.grad.copy_(torch.from_numpy(acc / self.gb))
        self.losses.append(tot)
        return tot

    def grad_tensor(self):
        return self.grad

    def apply_update(self):
        self.v.mul_(self.mu).add_(self.grad)
        self.p.sub_(self.lr * self.v)


def _case():
    from paper_1510_06706_b200 import configs as C
    cfg = C.scaled("c3", 10, (1, 1, 1), batch=4)
    rng = np.random.default_rng(3)
    params = C.init_params(cfg, 3).astype(np.float64)
    xs = [[rng.uniform(0, 1, size=cfg.in_dims)] for _ in range(cfg.batch)]
    labs = [[(rng.uniform(size=cfg.out_dims) < 0.5).astype(np.float64) for _ in range(3)]
            for _ in range(cfg.batch)]
    return cfg, params, xs, labs


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1510_06706_b200.distributed import DataParallelStep, shard_range
    cfg, params, xs, labs = _case()
    g = O.parse_netspec(cfg.netspec(), cfg.out_dims)
    net = OracleNet(g, params, cfg.batch, cfg.lr, cfg.momentum, cfg.loss)
    step = DataParallelStep(net, world)
    lo, hi = shard_range(cfg.batch, world, rank)
    for _ in range(2):
        step(xs[lo:hi], labs[lo:hi])
    out[rank] = net.p.numpy().copy()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_range():
    from paper_1510_06706_b200.distributed import shard_range
    assert [shard_range(16, 4, r) for r in range(4)] == [(0, 4), (4, 8), (8, 12), (12, 16)]
    with pytest.raises(ValueError):
        shard_range(10, 4, 0)


def test_gloo_world2_matches_full_batch():
    cfg, params, xs, labs = _case()
    g = O.parse_netspec(cfg.netspec(), cfg.out_dims)
    p, v = params.copy(), np.zeros(params.size)
    for _ in range(2):
        _, _, p, v = O.train_step(g, p, v, xs, labs, cfg.lr, cfg.momentum, cfg.loss)
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        assert np.max(np.abs(out[r] - p)) < 1e-12
    assert np.array_equal(out[0], out[1])
