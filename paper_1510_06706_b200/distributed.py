"""Data-parallel training over independent patches.

One process per GPU. A global batch of B patches is sharded B/N per rank;
each rank runs forward + loss + backward on its shard through the C-ABI
executor (gradients already scaled by 1/B_global), the flat gradient
buffer is summed across ranks with one NCCL allreduce (torch.distributed
is the plumbing; the gradient buffer is the executor's own device memory,
wrapped without a copy), then every rank applies the identical fused
SGD+momentum update. The reference has no distributed mode (SPEC.md:15,
650); at N=1 this is exactly its per-round update.

The step logic only needs an object with ``forward_backward``,
``grad_tensor`` and ``apply_update``, so the same code is exercised on CPU
(gloo, world size 2) by tests/test_distributed_cpu.py with an
oracle-backed stand-in.
"""
from __future__ import annotations


def shard_range(global_batch: int, world: int, rank: int):
    """Contiguous shard of patch indices for this rank (strong scaling)."""
    if global_batch % world:
        raise ValueError(f"global batch {global_batch} not divisible by {world} ranks")
    per = global_batch // world
    return rank * per, (rank + 1) * per


class DataParallelStep:
    """comm: the library's NCCL communicator (paper_1510_06706_b200.Comm):
    the step is then znn_net_train_step_dp (one allreduce per layer, issued
    as soon as that layer's gradient is final, on a communication stream
    overlapping the remaining backward). Without it the flat gradient buffer
    is summed with one torch.distributed allreduce (the gloo CPU tests)."""

    def __init__(self, net, world: int = 1, group=None, comm=None):
        self.net = net
        self.world = world
        self.group = group
        self.comm = comm
        self._grad = None

    def grad(self):
        if self._grad is None:
            self._grad = self.net.grad_tensor()
        return self._grad

    def __call__(self, inputs, labels, sync_loss=False):
        if self.world == 1 and hasattr(self.net, "train_step"):
            # nothing to sum: the update is fused into the backward pass
            return self.net.train_step(inputs, labels, sync_loss=sync_loss)
        if self.comm is not None:
            return self.net.train_step_dp(self.comm, inputs, labels, sync_loss=sync_loss)
        loss = self.net.forward_backward(inputs, labels, sync_loss=sync_loss)
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(self.grad(), op=dist.ReduceOp.SUM, group=self.group)
        self.net.apply_update()
        return loss
