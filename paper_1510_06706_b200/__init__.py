"""B200-native (sm_100a) ZNN training hot path (arXiv 1510.06706).

Public surface:
  Context, Net          -- device context and the per-rank network executor
  ops                   -- per-layer operators on CUDA tensors
  configs               -- the five BASELINE configurations as netspecs
  distributed           -- data-parallel training step (torch.distributed)
"""
from . import configs  # noqa: F401
from ._lib import ShapeError, ZnnError, lib  # noqa: F401
from .api import Context, Net, ops  # noqa: F401

__all__ = ["Context", "Net", "ops", "configs", "ShapeError", "ZnnError", "lib"]
