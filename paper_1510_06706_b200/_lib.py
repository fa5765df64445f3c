"""ctypes binding of libznn_cuda.so (include/znn_cuda.h).

The product path has no CPU fallback: if the shared library is missing, or
no sm_100 device is present, calls fail loudly (ZnnError)."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libznn_cuda.so")

ZNN_OK, ZNN_ERR_SHAPE, ZNN_ERR_RUNTIME = 0, 1, 2
ACT = {"logistic": 0, "sigmoid": 0, "tanh": 1, "relu": 2, "none": 3}
ENGINE = {"direct": 0, "fft": 1, "auto": 2, "simt": 3}
LOSS = {"l2": 0, "ce": 1}

# every symbol include/znn_cuda.h declares (checked by tests/test_capi_symbols.py)
EXPORTS = [
    "znn_version", "znn_device_count", "znn_ctx_create", "znn_ctx_destroy",
    "znn_ctx_set_stream", "znn_ctx_synchronize", "znn_last_error", "znn_ctx_launch_count",
    "znn_malloc", "znn_free", "znn_memcpy_h2d", "znn_memcpy_d2h",
    "znn_conv_fwd", "znn_conv_dgrad", "znn_conv_wgrad", "znn_transfer_fwd", "znn_transfer_bwd",
    "znn_maxpool_fwd", "znn_maxpool_bwd", "znn_maxfilter_fwd", "znn_maxfilter_bwd",
    "znn_loss", "znn_sgd_momentum",
    "znn_net_create", "znn_net_destroy", "znn_net_describe", "znn_net_num_params",
    "znn_net_io_sizes", "znn_net_set_params", "znn_net_get_params", "znn_net_get_gradients",
    "znn_net_reset_momentum", "znn_net_set_layer_engine", "znn_net_autotune", "znn_net_fft_counts",
    "znn_net_step_host", "znn_net_forward_backward", "znn_net_apply_update", "znn_net_train_step",
    "znn_net_grad_buffer", "znn_net_forward", "znn_net_group_info",
    "znn_net_get_group_image", "znn_net_get_mask", "znn_fft_cmac_time", "znn_fma_peak_tflops",
    "znn_fft_plan_create", "znn_fft_plan_destroy", "znn_fft_plan_info", "znn_fft_conv_fwd",
    "znn_fft_conv_bwd", "znn_fft_plan_counts", "znn_autotune_layer",
    "znn_comm_unique_id", "znn_comm_create", "znn_comm_destroy", "znn_allreduce", "znn_net_train_step_dp",
    "znn_net_set_graph", "znn_net_graph_captured", "znn_mem_stats",
    "znn_volume_write", "znn_volume_read", "znn_loader_open_dir", "znn_loader_open_host",
    "znn_loader_size", "znn_loader_destroy", "znn_net_step_loader", "znn_profile_enable", "znn_profile_report",
]


class ZnnError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


class ShapeError(ZnnError):
    """Reference structural_error (types.hpp:57-74)."""


class TrainCfg(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int64), ("global_batch", ctypes.c_int64),
                ("learning_rate", ctypes.c_float), ("momentum", ctypes.c_float),
                ("loss", ctypes.c_int), ("engine", ctypes.c_int), ("sliding", ctypes.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ZnnError(ZNN_ERR_RUNTIME, f"{LIB_PATH} is not built (run __graft_entry__.build()); "
                                        "there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, f32, i32, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_float, ctypes.c_int32, ctypes.c_int
    P64 = ctypes.POINTER(ctypes.c_int64)
    P32 = ctypes.POINTER(ctypes.c_int32)
    Pf = ctypes.POINTER(ctypes.c_float)
    Pd = ctypes.POINTER(ctypes.c_double)
    sig = {
        "znn_version": (ctypes.c_char_p, []),
        "znn_device_count": (ci, []),
        "znn_ctx_create": (ci, [ci, ctypes.POINTER(vp)]),
        "znn_ctx_destroy": (ci, [vp]),
        "znn_ctx_set_stream": (ci, [vp, vp]),
        "znn_ctx_synchronize": (ci, [vp]),
        "znn_last_error": (ctypes.c_char_p, [vp]),
        "znn_ctx_launch_count": (i64, [vp]),
        "znn_malloc": (ci, [vp, ctypes.c_size_t, ctypes.POINTER(vp)]),
        "znn_free": (ci, [vp, vp]),
        "znn_memcpy_h2d": (ci, [vp, vp, vp, ctypes.c_size_t]),
        "znn_memcpy_d2h": (ci, [vp, vp, vp, ctypes.c_size_t]),
        "znn_conv_fwd": (ci, [vp, vp, i64, i64, P64, vp, i64, P64, P64, vp, ci, vp, ci]),
        "znn_conv_dgrad": (ci, [vp, vp, i64, i64, P64, vp, i64, P64, P64, vp, ci]),
        "znn_conv_wgrad": (ci, [vp, vp, i64, i64, P64, vp, i64, P64, P64, vp, f32, ci]),
        "znn_transfer_fwd": (ci, [vp, vp, i64, i64, i64, P32, vp, vp]),
        "znn_transfer_bwd": (ci, [vp, vp, vp, ci, i64, i64, i64, P32, vp, vp, vp]),
        "znn_maxpool_fwd": (ci, [vp, vp, i64, P64, P64, vp, vp]),
        "znn_maxpool_bwd": (ci, [vp, vp, vp, i64, P64, P64, vp]),
        "znn_maxfilter_fwd": (ci, [vp, vp, i64, P64, P64, P64, vp, vp]),
        "znn_maxfilter_bwd": (ci, [vp, vp, vp, i64, P64, P64, P64, vp]),
        "znn_loss": (ci, [vp, ci, vp, vp, i64, f32, vp, Pd]),
        "znn_sgd_momentum": (ci, [vp, vp, vp, vp, i64, f32, f32]),
        "znn_net_create": (ci, [vp, ctypes.c_char_p, P64, ctypes.POINTER(TrainCfg), ctypes.POINTER(vp)]),
        "znn_net_destroy": (ci, [vp]),
        "znn_net_describe": (ctypes.c_char_p, [vp]),
        "znn_net_num_params": (ci, [vp, P64]),
        "znn_net_io_sizes": (ci, [vp, P64, P64]),
        "znn_net_set_params": (ci, [vp, Pf]),
        "znn_net_get_params": (ci, [vp, Pf]),
        "znn_net_get_gradients": (ci, [vp, Pf]),
        "znn_net_reset_momentum": (ci, [vp]),
        "znn_net_set_layer_engine": (ci, [vp, ci, ci]),
        "znn_net_autotune": (ci, [vp, ci, P32, ci]),
        "znn_net_fft_counts": (ci, [vp, ci, P64]),
        "znn_net_step_host": (ci, [vp, vp, vp, Pd]),
        "znn_net_forward_backward": (ci, [vp, vp, vp, Pd]),
        "znn_net_apply_update": (ci, [vp]),
        "znn_net_train_step": (ci, [vp, vp, vp, Pd]),
        "znn_net_grad_buffer": (ci, [vp, ctypes.POINTER(vp), P64]),
        "znn_net_forward": (ci, [vp, vp, Pf]),
        "znn_net_group_info": (ci, [vp, ci, P64, P64]),
        "znn_net_get_group_image": (ci, [vp, ci, ci, Pf]),
        "znn_net_get_mask": (ci, [vp, ci, P32]),
        "znn_fft_cmac_time": (ci, [vp, ci, i64, i64, i64, P64, P64, P64, ci, Pf, P64]),
        "znn_fma_peak_tflops": (ci, [vp, Pf]),
        "znn_fft_plan_create": (ci, [vp, i64, i64, i64, P64, P64, P64, ctypes.POINTER(vp)]),
        "znn_fft_plan_destroy": (ci, [vp]),
        "znn_fft_plan_info": (ci, [vp, P64, P64, P64]),
        "znn_fft_conv_fwd": (ci, [vp, vp, vp, vp, ci, vp]),
        "znn_fft_conv_bwd": (ci, [vp, vp, vp, vp, vp]),
        "znn_fft_plan_counts": (ci, [vp, P64]),
        "znn_autotune_layer": (ci, [vp, i64, i64, i64, P64, P64, P64, ci, ctypes.POINTER(ci), Pf]),
        "znn_comm_unique_id": (ci, [vp]),
        "znn_comm_create": (ci, [vp, vp, ci, ci, ctypes.POINTER(vp)]),
        "znn_comm_destroy": (ci, [vp]),
        "znn_allreduce": (ci, [vp, vp, i64]),
        "znn_net_train_step_dp": (ci, [vp, vp, vp, vp, Pd]),
        "znn_net_set_graph": (ci, [vp, ci]),
        "znn_net_graph_captured": (ci, [vp, ctypes.POINTER(ci)]),
        "znn_mem_stats": (ci, [vp, P64]),
        "znn_volume_write": (ci, [ctypes.c_char_p, P64, vp]),
        "znn_volume_read": (ci, [ctypes.c_char_p, P64, vp, i64]),
        "znn_loader_open_dir": (ci, [vp, ctypes.c_char_p, i64, ctypes.POINTER(vp)]),
        "znn_loader_open_host": (ci, [vp, vp, vp, i64, i64, ctypes.POINTER(vp)]),
        "znn_loader_size": (ci, [vp, P64]),
        "znn_loader_destroy": (ci, [vp]),
        "znn_net_step_loader": (ci, [vp, vp, Pd]),
        "znn_profile_enable": (ci, [vp, ci]),
        "znn_profile_report": (ci, [vp, ctypes.c_char_p, i64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(status, ctx=None):
    if status == ZNN_OK:
        return
    msg = lib().znn_last_error(ctx).decode(errors="replace")
    if status == ZNN_ERR_SHAPE:
        raise ShapeError(status, msg)
    raise ZnnError(status, msg)


def v3(t):
    return (ctypes.c_int64 * 3)(*[int(v) for v in t])
