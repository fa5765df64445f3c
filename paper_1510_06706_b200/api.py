"""Python host API over libznn_cuda.so.

Mirrors the reference's host surface for this path:
  * ``Net`` <-> ``net_graph`` + ``engine<float>`` + ``train`` (netgraph.hpp,
    engine.hpp:65-295, trainer.hpp:265-318): built from netspec text, flat
    parameters in the reference's edge-id order, one SGD step per call;
  * ``ops`` functions <-> conv_direct.hpp / maxops.hpp / transfer.hpp free
    functions, but per layer and per batch on CUDA tensors.
torch is used only for device memory and streams (plumbing).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import ACT, ENGINE, LOSS, check, lib, v3


def _ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _fptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


class Context:
    """znn_ctx: one CUDA device + the stream all work is queued on."""

    def __init__(self, device: int = 0, stream=None):
        self._h = ctypes.c_void_p()
        check(lib().znn_ctx_create(int(device), ctypes.byref(self._h)))
        self.device = device
        if stream is not None:
            self.set_stream(stream)

    def set_stream(self, stream):
        """stream: a torch.cuda.Stream or a raw cudaStream_t integer."""
        handle = getattr(stream, "cuda_stream", stream)
        check(lib().znn_ctx_set_stream(self._h, ctypes.c_void_p(int(handle))), self._h)

    def synchronize(self):
        check(lib().znn_ctx_synchronize(self._h), self._h)

    def launches(self) -> int:
        return int(lib().znn_ctx_launch_count(self._h))

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            lib().znn_ctx_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Net:
    """GPU executor for one data-parallel rank (engine<float> + train step)."""

    def __init__(self, ctx: Context, netspec: str, out_dims=None, batch=1, global_batch=None,
                 lr=0.01, momentum=0.0, loss="l2", engine="direct", sliding=False):
        self.ctx = ctx
        cfg = _lib.TrainCfg(int(batch), int(global_batch or batch), float(lr), float(momentum),
                            LOSS[loss], ENGINE[engine], 1 if sliding else 0)
        self._h = ctypes.c_void_p()
        od = v3(out_dims) if out_dims is not None else None
        check(lib().znn_net_create(ctx.handle, netspec.encode(), od, ctypes.byref(cfg),
                                   ctypes.byref(self._h)), ctx.handle)
        self.batch = int(batch)
        n = ctypes.c_int64()
        check(lib().znn_net_num_params(self._h, ctypes.byref(n)), ctx.handle)
        self.num_params = n.value
        a, b = ctypes.c_int64(), ctypes.c_int64()
        check(lib().znn_net_io_sizes(self._h, ctypes.byref(a), ctypes.byref(b)), ctx.handle)
        self.in_per_patch, self.out_per_patch = a.value, b.value
        if engine == "auto":
            self.autotune()

    def _c(self, st):
        check(st, self.ctx.handle)

    def describe(self) -> str:
        return lib().znn_net_describe(self._h).decode()

    def set_params(self, p):
        p = np.ascontiguousarray(p, dtype=np.float32)
        assert p.size == self.num_params, (p.size, self.num_params)
        self._c(lib().znn_net_set_params(self._h, _fptr(p)))

    def get_params(self) -> np.ndarray:
        out = np.empty(self.num_params, dtype=np.float32)
        self._c(lib().znn_net_get_params(self._h, _fptr(out)))
        return out

    def get_gradients(self) -> np.ndarray:
        out = np.empty(self.num_params, dtype=np.float32)
        self._c(lib().znn_net_get_gradients(self._h, _fptr(out)))
        return out

    def reset_momentum(self):
        self._c(lib().znn_net_reset_momentum(self._h))

    def set_layer_engine(self, conv_layer: int, engine: str):
        self._c(lib().znn_net_set_layer_engine(self._h, conv_layer, ENGINE[engine]))

    def autotune(self, trials: int = 3):
        arr = (ctypes.c_int32 * 64)()
        self._c(lib().znn_net_autotune(self._h, trials, arr, 64))
        nconv = sum(1 for ln in self.describe().splitlines() if "conv#" in ln and not ln.startswith("autotune"))
        self.engines = [int(v) for v in arr[:nconv]]
        return self.engines

    def fft_counts(self, conv_layer: int):
        """FFT transform counters (fwd/bwd/upd x image/kernel/inverse) of a conv layer."""
        out = (ctypes.c_int64 * 9)()
        self._c(lib().znn_net_fft_counts(self._h, conv_layer, out))
        keys = [f"{p}_{k}" for p in ("fwd", "bwd", "upd") for k in ("image", "kernel", "inverse")]
        return dict(zip(keys, [int(v) for v in out]))

    def step_host(self, inputs: np.ndarray, labels: np.ndarray) -> float:
        """One SGD step from HOST arrays (H2D, fwd, loss, bwd, update, loss D2H)."""
        inputs = np.ascontiguousarray(inputs, dtype=np.float32)
        labels = np.ascontiguousarray(labels, dtype=np.float32)
        assert inputs.size == self.batch * self.in_per_patch
        assert labels.size == self.batch * self.out_per_patch
        loss = ctypes.c_double()
        self._c(lib().znn_net_step_host(self._h, inputs.ctypes.data_as(ctypes.c_void_p),
                                        labels.ctypes.data_as(ctypes.c_void_p), ctypes.byref(loss)))
        return loss.value

    def step_host_ptr(self, in_ptr: int, lab_ptr: int) -> float:
        loss = ctypes.c_double()
        self._c(lib().znn_net_step_host(self._h, ctypes.c_void_p(in_ptr), ctypes.c_void_p(lab_ptr),
                                        ctypes.byref(loss)))
        return loss.value

    def forward_backward(self, inputs_dev, labels_dev, sync_loss=True):
        """inputs_dev / labels_dev: CUDA tensors (or raw device pointers)."""
        ip = inputs_dev if isinstance(inputs_dev, int) else inputs_dev.data_ptr()
        lp = labels_dev if isinstance(labels_dev, int) else labels_dev.data_ptr()
        if sync_loss:
            loss = ctypes.c_double()
            self._c(lib().znn_net_forward_backward(self._h, ctypes.c_void_p(ip), ctypes.c_void_p(lp),
                                                   ctypes.byref(loss)))
            return loss.value
        self._c(lib().znn_net_forward_backward(self._h, ctypes.c_void_p(ip), ctypes.c_void_p(lp), None))
        return None

    def train_step(self, inputs_dev, labels_dev, sync_loss=True):
        """One SGD step from device buffers with the update fused layer by
        layer (single process; = forward_backward + apply_update)."""
        ip = inputs_dev if isinstance(inputs_dev, int) else inputs_dev.data_ptr()
        lp = labels_dev if isinstance(labels_dev, int) else labels_dev.data_ptr()
        if sync_loss:
            loss = ctypes.c_double()
            self._c(lib().znn_net_train_step(self._h, ctypes.c_void_p(ip), ctypes.c_void_p(lp), ctypes.byref(loss)))
            return loss.value
        self._c(lib().znn_net_train_step(self._h, ctypes.c_void_p(ip), ctypes.c_void_p(lp), None))
        return None

    def apply_update(self):
        self._c(lib().znn_net_apply_update(self._h))

    def grad_buffer(self):
        """(device pointer, length) of the flat gradient buffer."""
        p, n = ctypes.c_void_p(), ctypes.c_int64()
        self._c(lib().znn_net_grad_buffer(self._h, ctypes.byref(p), ctypes.byref(n)))
        return p.value, n.value

    def grad_tensor(self):
        """The flat gradient buffer as a torch CUDA tensor view (no copy)."""
        import torch
        ptr, n = self.grad_buffer()

        class _Iface:
            __cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                        "version": 3, "strides": None}

        return torch.as_tensor(_Iface(), device=f"cuda:{self.ctx.device}")

    def forward(self, inputs_dev) -> np.ndarray:
        out = np.empty(self.batch * self.out_per_patch, dtype=np.float32)
        ip = inputs_dev if isinstance(inputs_dev, int) else inputs_dev.data_ptr()
        self._c(lib().znn_net_forward(self._h, ctypes.c_void_p(ip), _fptr(out)))
        return out

    def set_graph(self, on=True):
        """CUDA-graph mode for train_step / step_host / step_loader (the first
        step eager, then one captured graph per input buffer pair)."""
        self._c(lib().znn_net_set_graph(self._h, 1 if on else 0))

    def graph_captured(self) -> bool:
        v = ctypes.c_int()
        self._c(lib().znn_net_graph_captured(self._h, ctypes.byref(v)))
        return bool(v.value)

    def train_step_dp(self, comm, inputs_dev, labels_dev, sync_loss=True):
        """Data-parallel step: per-layer NCCL allreduce overlapped with the backward, then the update."""
        ip = inputs_dev if isinstance(inputs_dev, int) else inputs_dev.data_ptr()
        lp = labels_dev if isinstance(labels_dev, int) else labels_dev.data_ptr()
        loss = ctypes.c_double()
        self._c(lib().znn_net_train_step_dp(self._h, comm.handle, ctypes.c_void_p(ip), ctypes.c_void_p(lp),
                                            ctypes.byref(loss) if sync_loss else None))
        return loss.value if sync_loss else None

    def step_loader(self, loader) -> float:
        loss = ctypes.c_double()
        self._c(lib().znn_net_step_loader(self._h, loader.handle, ctypes.byref(loss)))
        return loss.value

    def group_info(self, g):
        maps, d = ctypes.c_int64(), (ctypes.c_int64 * 3)()
        self._c(lib().znn_net_group_info(self._h, g, ctypes.byref(maps), d))
        return maps.value, tuple(d)

    def group_image(self, g, which=0) -> np.ndarray:
        maps, d = self.group_info(g)
        out = np.empty((self.batch, abs(maps)) + d, dtype=np.float32)
        self._c(lib().znn_net_get_group_image(self._h, g, which, _fptr(out)))
        return out

    def group_mask(self, g) -> np.ndarray:
        maps, d = self.group_info(g)
        out = np.empty((self.batch, abs(maps)) + d, dtype=np.int32)
        self._c(lib().znn_net_get_mask(self._h, g, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
        return out

    def close(self):
        if self._h:
            lib().znn_net_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# per-layer operators on torch CUDA tensors ([B][maps][x][y][z] fp32)
# ---------------------------------------------------------------------------

class ops:
    @staticmethod
    def conv_fwd(ctx, x, w, k, s=(1, 1, 1), bias=None, act="none", engine="direct"):
        import torch
        B, f_in = x.shape[0], x.shape[1]
        n = tuple(x.shape[2:])
        f_out = w.shape[0]
        m = tuple(n[a] - s[a] * (k[a] - 1) for a in range(3))
        y = torch.empty((B, f_out) + m, device=x.device, dtype=torch.float32)
        check(lib().znn_conv_fwd(ctx.handle, _ptr(x), B, f_in, v3(n), _ptr(w), f_out, v3(k), v3(s),
                                 _ptr(bias), ACT[act], _ptr(y), ENGINE[engine]), ctx.handle)
        return y

    @staticmethod
    def conv_dgrad(ctx, g, w, k, s=(1, 1, 1), engine="direct"):
        import torch
        B, f_out = g.shape[0], g.shape[1]
        m = tuple(g.shape[2:])
        f_in = w.shape[1]
        n = tuple(m[a] + s[a] * (k[a] - 1) for a in range(3))
        dx = torch.empty((B, f_in) + n, device=g.device, dtype=torch.float32)
        check(lib().znn_conv_dgrad(ctx.handle, _ptr(g), B, f_out, v3(m), _ptr(w), f_in, v3(k), v3(s),
                                   _ptr(dx), ENGINE[engine]), ctx.handle)
        return dx

    @staticmethod
    def conv_wgrad(ctx, x, g, k, s=(1, 1, 1), scale=1.0, engine="direct"):
        import torch
        B, f_in = x.shape[0], x.shape[1]
        n = tuple(x.shape[2:])
        f_out = g.shape[1]
        dw = torch.empty((f_out, f_in) + tuple(k), device=x.device, dtype=torch.float32)
        check(lib().znn_conv_wgrad(ctx.handle, _ptr(x), B, f_in, v3(n), _ptr(g), f_out, v3(k), v3(s),
                                   _ptr(dw), float(scale), ENGINE[engine]), ctx.handle)
        return dw

    @staticmethod
    def transfer_fwd(ctx, x, kinds, bias=None):
        import torch
        B, f = x.shape[0], x.shape[1]
        vox = int(np.prod(x.shape[2:]))
        kd = (ctypes.c_int32 * f)(*[ACT[k] if isinstance(k, str) else int(k) for k in kinds])
        y = torch.empty_like(x)
        check(lib().znn_transfer_fwd(ctx.handle, _ptr(x), B, f, vox, kd, _ptr(bias), _ptr(y)), ctx.handle)
        return y

    @staticmethod
    def transfer_bwd(ctx, g, xy, kinds, bias=None, from_output=False, want_dbias=True):
        import torch
        B, f = g.shape[0], g.shape[1]
        vox = int(np.prod(g.shape[2:]))
        kd = (ctypes.c_int32 * f)(*[ACT[k] if isinstance(k, str) else int(k) for k in kinds])
        gx = torch.empty_like(g)
        db = torch.empty(f, device=g.device, dtype=torch.float32) if want_dbias else None
        check(lib().znn_transfer_bwd(ctx.handle, _ptr(g), _ptr(xy), 1 if from_output else 0, B, f, vox, kd,
                                     _ptr(bias), _ptr(gx), _ptr(db)), ctx.handle)
        return gx, db

    @staticmethod
    def maxpool_fwd(ctx, x, p):
        import torch
        lead = x.shape[:-3]
        n = tuple(x.shape[-3:])
        maps = int(np.prod(lead)) if lead else 1
        m = tuple(n[a] // p[a] for a in range(3))
        y = torch.empty(tuple(lead) + m, device=x.device, dtype=torch.float32)
        mask = torch.empty(tuple(lead) + m, device=x.device, dtype=torch.int32)
        check(lib().znn_maxpool_fwd(ctx.handle, _ptr(x), maps, v3(n), v3(p), _ptr(y), _ptr(mask)), ctx.handle)
        return y, mask

    @staticmethod
    def maxpool_bwd(ctx, g, mask, p):
        import torch
        lead = g.shape[:-3]
        m = tuple(g.shape[-3:])
        maps = int(np.prod(lead)) if lead else 1
        dx = torch.empty(tuple(lead) + tuple(m[a] * p[a] for a in range(3)), device=g.device,
                         dtype=torch.float32)
        check(lib().znn_maxpool_bwd(ctx.handle, _ptr(g), _ptr(mask), maps, v3(m), v3(p), _ptr(dx)), ctx.handle)
        return dx

    @staticmethod
    def maxfilter_fwd(ctx, x, k, s=(1, 1, 1)):
        import torch
        lead = x.shape[:-3]
        n = tuple(x.shape[-3:])
        maps = int(np.prod(lead)) if lead else 1
        m = tuple(n[a] - s[a] * (k[a] - 1) for a in range(3))
        y = torch.empty(tuple(lead) + m, device=x.device, dtype=torch.float32)
        mask = torch.empty(tuple(lead) + m, device=x.device, dtype=torch.int32)
        check(lib().znn_maxfilter_fwd(ctx.handle, _ptr(x), maps, v3(n), v3(k), v3(s), _ptr(y), _ptr(mask)),
              ctx.handle)
        return y, mask

    @staticmethod
    def maxfilter_bwd(ctx, g, mask, k, s=(1, 1, 1)):
        import torch
        lead = g.shape[:-3]
        m = tuple(g.shape[-3:])
        maps = int(np.prod(lead)) if lead else 1
        n = tuple(m[a] + s[a] * (k[a] - 1) for a in range(3))
        dx = torch.empty(tuple(lead) + n, device=g.device, dtype=torch.float32)
        check(lib().znn_maxfilter_bwd(ctx.handle, _ptr(g), _ptr(mask), maps, v3(m), v3(k), v3(s), _ptr(dx)),
              ctx.handle)
        return dx

    @staticmethod
    def loss(ctx, kind, a, d, scale=1.0):
        import torch
        grad = torch.empty_like(a)
        out = ctypes.c_double()
        check(lib().znn_loss(ctx.handle, LOSS[kind], _ptr(a), _ptr(d), a.numel(), float(scale), _ptr(grad),
                             ctypes.byref(out)), ctx.handle)
        return out.value, grad

    @staticmethod
    def sgd_momentum(ctx, w, v, g, lr, mu):
        check(lib().znn_sgd_momentum(ctx.handle, _ptr(w), _ptr(v), _ptr(g), w.numel(), float(lr), float(mu)),
              ctx.handle)

    @staticmethod
    def fft_cmac_time(ctx, which, B, f_in, f_out, n, k, s=(1, 1, 1), reps=3):
        """(average device ms, bins) of one FFT-engine CMAC launch (0 fwd,
        1 data gradient, 2 kernel-gradient product) for a conv layer shape,
        on synthetic spectra."""
        ms, bins = ctypes.c_float(), ctypes.c_int64()
        check(lib().znn_fft_cmac_time(ctx.handle, int(which), int(B), int(f_in), int(f_out), v3(n), v3(k), v3(s),
                                      int(reps), ctypes.byref(ms), ctypes.byref(bins)), ctx.handle)
        return ms.value, bins.value

    @staticmethod
    def fma_peak_tflops(ctx):
        """Measured FP32 FMA throughput of the device (TFLOP/s)."""
        t = ctypes.c_float()
        check(lib().znn_fma_peak_tflops(ctx.handle, ctypes.byref(t)), ctx.handle)
        return t.value



def mem_stats(ctx: Context) -> dict:
    """Device free/total bytes and the library's own device allocations so far."""
    out = (ctypes.c_int64 * 4)()
    check(lib().znn_mem_stats(ctx.handle, out), ctx.handle)
    return {"free": int(out[0]), "total": int(out[1]), "allocs": int(out[2]), "alloc_bytes": int(out[3])}


class FftPlan:
    """FFT engine for one fully connected layer (fft_plan_cache + memo_store,
    fft.hpp:57-192 / conv_fft.hpp:127-192): forward memoises the image and
    kernel spectra; backward gives dx (optional) and dw from that memo."""

    def __init__(self, ctx: Context, B, f_in, f_out, n, k, s=(1, 1, 1)):
        self.ctx = ctx
        self.B, self.f_in, self.f_out = int(B), int(f_in), int(f_out)
        self.n, self.k, self.s = tuple(n), tuple(k), tuple(s)
        self.m = tuple(self.n[a] - self.s[a] * (self.k[a] - 1) for a in range(3))
        self._h = ctypes.c_void_p()
        check(lib().znn_fft_plan_create(ctx.handle, self.B, self.f_in, self.f_out, v3(n), v3(k), v3(s),
                                        ctypes.byref(self._h)), ctx.handle)

    def info(self):
        pads, bins, kb = (ctypes.c_int64 * 3)(), ctypes.c_int64(), ctypes.c_int64()
        check(lib().znn_fft_plan_info(self._h, pads, ctypes.byref(bins), ctypes.byref(kb)), self.ctx.handle)
        return {"pads": tuple(pads), "bins": bins.value, "kernel_spectrum_bytes": kb.value}

    def forward(self, x, w, bias=None, act="none"):
        import torch
        y = torch.empty((self.B, self.f_out) + self.m, device=x.device, dtype=torch.float32)
        check(lib().znn_fft_conv_fwd(self._h, _ptr(x), _ptr(w), _ptr(bias), ACT[act], _ptr(y)), self.ctx.handle)
        return y

    def backward(self, g, w, want_dx=True):
        import torch
        dw = torch.empty((self.f_out, self.f_in) + self.k, device=g.device, dtype=torch.float32)
        dx = torch.empty((self.B, self.f_in) + self.n, device=g.device, dtype=torch.float32) if want_dx else None
        check(lib().znn_fft_conv_bwd(self._h, _ptr(g), _ptr(w), _ptr(dw), _ptr(dx)), self.ctx.handle)
        return dx, dw

    def counts(self):
        out = (ctypes.c_int64 * 9)()
        check(lib().znn_fft_plan_counts(self._h, out), self.ctx.handle)
        keys = [f"{p}_{k}" for p in ("fwd", "bwd", "upd") for k in ("image", "kernel", "inverse")]
        return dict(zip(keys, [int(v) for v in out]))

    def close(self):
        if self._h:
            lib().znn_fft_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def autotune_layer(ctx: Context, B, f_in, f_out, n, k, s=(1, 1, 1), trials=3):
    """Per-layer engine choice by device timing (autotune_modes, trainer.hpp:181-250):
    returns (engine name, {engine: median ms of fwd+dgrad+wgrad})."""
    chosen = ctypes.c_int()
    ms = (ctypes.c_float * 3)()
    check(lib().znn_autotune_layer(ctx.handle, int(B), int(f_in), int(f_out), v3(n), v3(k), v3(s), int(trials),
                                   ctypes.byref(chosen), ms), ctx.handle)
    names = {0: "direct", 1: "fft", 3: "simt"}
    times = {nm: float(ms[i]) for i, nm in enumerate(("direct", "fft", "simt")) if ms[i] >= 0}
    return names[chosen.value], times


class Comm:
    """NCCL communicator of one rank (znn_comm); the 128-byte id comes from
    comm_unique_id() on rank 0 and is shared by the caller."""

    def __init__(self, ctx: Context, unique_id: bytes, nranks: int, rank: int):
        self.ctx = ctx
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        self._h = ctypes.c_void_p()
        check(lib().znn_comm_create(ctx.handle, buf, int(nranks), int(rank), ctypes.byref(self._h)), ctx.handle)

    @property
    def handle(self):
        return self._h

    def allreduce(self, t):
        check(lib().znn_allreduce(self._h, _ptr(t), t.numel()), self.ctx.handle)

    def close(self):
        if self._h:
            lib().znn_comm_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(lib().znn_comm_unique_id(buf))
    return buf.raw


def write_volume(path: str, vol: np.ndarray):
    """ZNNV file (volume_io.hpp:15-86) from a 3-D float array (x-major)."""
    v = np.ascontiguousarray(vol, dtype=np.float32)
    assert v.ndim == 3
    check(lib().znn_volume_write(path.encode(), v3(v.shape), v.ctypes.data_as(ctypes.c_void_p)))


def read_volume(path: str) -> np.ndarray:
    d = (ctypes.c_int64 * 3)()
    check(lib().znn_volume_read(path.encode(), d, None, 0))
    out = np.empty(tuple(d), dtype=np.float32)
    check(lib().znn_volume_read(path.encode(), d, out.ctypes.data_as(ctypes.c_void_p), out.size))
    return out


class Loader:
    """Data provider (trainer.hpp:87-166) with pinned double-buffered H2D:
    from a directory (inputs/ + labels/ ZNNV files) or host arrays."""

    def __init__(self, net: Net, directory: str = None, inputs=None, labels=None, shard_offset: int = 0):
        self.net = net
        self._h = ctypes.c_void_p()
        self._keep = None
        if directory is not None:
            check(lib().znn_loader_open_dir(net._h, directory.encode(), int(shard_offset), ctypes.byref(self._h)),
                  net.ctx.handle)
        else:
            ip = inputs.data_ptr() if hasattr(inputs, "data_ptr") else inputs.ctypes.data
            lp = labels.data_ptr() if hasattr(labels, "data_ptr") else labels.ctypes.data
            samples = inputs.shape[0]
            self._keep = (inputs, labels)
            check(lib().znn_loader_open_host(net._h, ctypes.c_void_p(ip), ctypes.c_void_p(lp), int(samples),
                                             int(shard_offset), ctypes.byref(self._h)), net.ctx.handle)

    @property
    def handle(self):
        return self._h

    def __len__(self):
        n = ctypes.c_int64()
        check(lib().znn_loader_size(self._h, ctypes.byref(n)))
        return n.value

    def close(self):
        if self._h:
            lib().znn_loader_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def profile_enable(ctx: Context, on=True):
    check(lib().znn_profile_enable(ctx.handle, 1 if on else 0), ctx.handle)


def profile_report(ctx: Context):
    """[{kernel, launches, ms, bytes, flops}] recorded since the last report."""
    import json
    buf = ctypes.create_string_buffer(1 << 20)
    check(lib().znn_profile_report(ctx.handle, buf, len(buf)), ctx.handle)
    return json.loads(buf.value.decode())
