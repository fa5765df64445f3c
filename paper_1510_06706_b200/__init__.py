"""B200-native (sm_100a) ZNN training hot path (arXiv 1510.06706).

Public surface:
  Context, Net          -- device context and the per-rank network executor
  ops                   -- per-layer operators on CUDA tensors
  configs               -- the five BASELINE configurations as netspecs
  FftPlan, autotune_layer -- the FFT engine and the autotuner per layer
  Comm, comm_unique_id  -- NCCL communicator for data parallelism
  Loader, read/write_volume -- data provider and ZNNV volume files
  distributed           -- data-parallel training step
"""
from . import configs  # noqa: F401
from ._lib import ShapeError, ZnnError, lib  # noqa: F401
from .api import (Comm, Context, FftPlan, Loader, Net, autotune_layer, comm_unique_id, mem_stats,  # noqa: F401
                  ops, read_volume, write_volume)

__all__ = ["Context", "Net", "ops", "configs", "ShapeError", "ZnnError", "lib", "FftPlan", "autotune_layer",
           "Comm", "comm_unique_id", "mem_stats", "Loader", "read_volume", "write_volume"]
