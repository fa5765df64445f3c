#!/usr/bin/env python
"""Benchmark: 3D ConvNet training output voxels/s (fwd + bwd + update).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

A step = one SGD+momentum step of the BASELINE config over its global batch
of synthetic patches (uniform[0,1) inputs, Bernoulli(0.5) labels, Glorot
weights from the seed). N>1 is launched by torchrun (one rank per GPU,
NCCL gradient allreduce, global batch sharded -> strong scaling).
Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default=os.environ.get("ZNN_BENCH_CONFIG", "c5"))
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--engine", default=None)
    p.add_argument("--e2e-steps", type=int, default=None)
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


# ---------------------------------------------------------------------------
# clocks sampled DURING the timed region (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and
                          r[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peaks():
    for p in (os.path.join(ROOT, "MEASURED_PEAKS.json"),):
        if os.path.exists(p):
            with open(p) as f:
                return json.load(f), "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
        "fallback (B200_PROFILING.md)"


def tf32_peak_tflops(torch):
    """cuBLAS TF32 dense GEMM 8192^3, best of 5 (the denominator for 3xTF32
    tensor-pipe utilisation; MEASURED_PEAKS.json carries bf16 only)."""
    torch.backends.cuda.matmul.allow_tf32 = True
    n = 8192
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    for _ in range(2):
        a @ b
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        a @ b
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    torch.backends.cuda.matmul.allow_tf32 = False
    del a, b
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


# ---------------------------------------------------------------------------
# CPU baseline (oracle/_ref reference engine if built, else the oracle port)
# ---------------------------------------------------------------------------
def cpu_baseline(cfg, budget_s=20.0):
    sys.path.insert(0, ROOT)
    from oracle import cpu_bench
    return cpu_bench.run(cfg, budget_s=budget_s)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_1510_06706_b200 import configs
    cfg = configs.CONFIGS[args.config]
    out_vox = int(np.prod(cfg.out_dims))
    vals = []
    cb = None
    for _ in range(args.steps):
        cb = cpu_baseline(cfg, budget_s=float(os.environ.get("ZNN_REF_BUDGET_S", "20")))
        vals.append(cb["value"])
    v = float(np.median(vals))
    cb["value"] = v
    line = {"metric": "train_output_voxels_per_s", "value": v, "unit": "voxels/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": out_vox * cfg.batch / v * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": cb.get("dtype", "f32"),
            "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg.name, "global_batch": cfg.batch, "in_dims": cfg.in_dims,
                       "out_dims": cfg.out_dims, "parallelism": "cpu threads"},
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "voxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1510_06706_b200 import Context, Net, configs, ops
    from paper_1510_06706_b200.distributed import DataParallelStep, shard_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        raise SystemExit(f"WORLD_SIZE={world} but --gpus {args.gpus}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    cfg = configs.CONFIGS[args.config]
    engine = args.engine or cfg.engine
    B = cfg.batch
    lo, hi = shard_range(B, world, rank)
    Bl = hi - lo
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = Context(local, stream)
    net = Net(ctx, cfg.netspec(), cfg.out_dims, batch=Bl, global_batch=B, lr=cfg.lr,
              momentum=cfg.momentum, loss=cfg.loss, engine=engine)
    net.set_params(configs.init_params(cfg, 2026))

    rng = np.random.default_rng(1000 + rank)
    n_out = cfg.layers[-1].width
    x_host = torch.from_numpy(rng.uniform(0, 1, size=(Bl, cfg.in_maps) + tuple(cfg.in_dims))
                              .astype(np.float32)).pin_memory()
    y_host = torch.from_numpy((rng.uniform(size=(Bl, n_out) + tuple(cfg.out_dims)) < 0.5)
                              .astype(np.float32)).pin_memory()
    x_dev = x_host.to("cuda", non_blocking=True)
    y_dev = y_host.to("cuda", non_blocking=True)
    torch.cuda.synchronize()
    step = DataParallelStep(net, world)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident timed region ----
    for _ in range(args.warmup):
        step(x_dev, y_dev)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            step(x_dev, y_dev)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches = ctx.launches() - launches0
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)

    out_vox = int(np.prod(cfg.out_dims))
    value = B * out_vox / (ms * 1e-3)

    # ---- end-to-end through the C-ABI with HOST buffers ----
    e2e_steps = args.e2e_steps or max(2, args.steps // 2)
    h2d = (x_host.numel() + y_host.numel()) * 4
    d2h = 8
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        if world == 1:
            net.step_host_ptr(x_host.data_ptr(), y_host.data_ptr())  # H2D, fwd, bwd, update, loss D2H
        else:
            x_dev.copy_(x_host, non_blocking=True)
            y_dev.copy_(y_host, non_blocking=True)
            step(x_dev, y_dev, sync_loss=True)
    e1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    e2e_ms = max_over_ranks(max(e0.elapsed_time(e1), wall * 1e3) / e2e_steps)
    e2e_value = B * out_vox / (e2e_ms * 1e-3)

    engines = list(getattr(net, "engines", []) or [])
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel of the largest conv layer, on the
    # engine that layer runs (the net's device memory is released first) ----
    net.close()
    torch.cuda.empty_cache()
    roof = dominant_kernel_roofline(torch, ctx, ops, cfg, Bl, engine, stream, engines)
    line = {
        "metric": "train_output_voxels_per_s", "value": value, "unit": "voxels/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg.name, "global_batch": B, "per_gpu_batch": Bl, "in_dims": cfg.in_dims,
                   "out_dims": cfg.out_dims, "parallelism": f"dp{world}", "engine": engine,
                   "conv_engines": [{0: "direct", 1: "fft", 3: "direct-simt"}.get(e, str(e)) for e in engines]
                   if engines else None,
                   "l2": "inputs larger than L2 (per-step working set >> 126 MB)",
                   "conv_tflops_per_step": configs.conv_flops_per_patch(cfg) * B / 1e12},
        "conv_tflops_algorithmic": configs.conv_flops_per_patch(cfg) * B / (ms * 1e-3) / 1e12,
        "e2e": {"value": e2e_value, "unit": "voxels/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
        "roofline": roof,
    }
    if not args.no_cpu_baseline and world == 1:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg, budget_s=float(os.environ.get("ZNN_CPU_BUDGET_S", "20")))
        except Exception as e:  # the baseline is reported, never the product path
            line["cpu_baseline"] = {"error": str(e)[:200]}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def fft_cmac_roofline(torch, ctx, ops, Bl, fi, fo, n, k, s):
    """The FFT engine's dominant kernel is the per-bin complex multiply-
    accumulate over converging edges. At B = 16 each kernel-
    spectrum element feeds 16 complex MACs (8 flop per 8 bytes), so it is
    bound by FP32 FMA issue, not HBM: the roofline is the measured FMA peak,
    with the HBM view (algorithmic bytes / time) beside it."""
    peaks, peak_src = measured_peaks()
    names = {0: "fwd", 1: "dgrad", 2: "upd"}
    times, bins = {}, None
    for which in (0, 1, 2):
        if which == 1 and fi == 1:
            continue
        ms, bins = ops.fft_cmac_time(ctx, which, Bl, fi, fo, n, k, s, reps=3)
        times[names[which]] = ms * 1e-3
    dom = max(times, key=times.get)
    dur = times[dom]
    flops = 8.0 * Bl * fi * fo * bins  # complex MAC = 4 FMA
    c8 = 8.0 * bins  # bytes per spectrum (complex64)
    byts = {"fwd": c8 * (fi * fo + Bl * fi + Bl * fo), "dgrad": c8 * (fi * fo + Bl * fo + Bl * fi),
            "upd": c8 * (Bl * fi + Bl * fo + fi * fo)}[dom]
    fma_peak = ops.fma_peak_tflops(ctx)
    achieved = flops / dur / 1e12
    shape = f"f={fi}->{fo} n={tuple(n)} k={tuple(k)} s={tuple(s)} B={Bl} bins={bins}"
    traffic, traffic_src = None, None
    import glob
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic_*.json"))):
        try:
            with open(f) as fh:
                cap = json.load(fh)
            if cap.get("shape") == "cmac " + shape and dom in cap.get("per_launch", {}):
                traffic = cap["per_launch"][dom]["dram_bytes"]
                traffic_src = os.path.relpath(f, ROOT) + " (ncu dram__bytes_read.sum + dram__bytes_write.sum)"
        except Exception:
            pass
    return {"bound": "fp32-fma", "kernel": f"fft_cmac_{dom} " + shape,
            "achieved": achieved, "peak": fma_peak, "unit": "TFLOP/s", "frac": achieved / fma_peak,
            "achieved_is": "algorithmic fp32 FLOP/s (8 B f f' bins per launch: complex MAC = 4 FMA) / "
                           "CUDA-event duration of the launch",
            "peak_source": "measured in-run: 3-register FP32 FFMA issue-rate probe (znn_fma_peak_tflops; "
                           "every CMAC FMA has three register operands; the immediate-operand form peaks at "
                           "71.9 TFLOP/s, tests/micro/mma_rate.cu); MEASURED_PEAKS.json has HBM and bf16 only",
            "hbm_view": {"algorithmic_bytes": byts, "achieved_gbs": byts / dur / 1e9,
                         "peak_gbs": peaks["hbm_gbs"], "frac": byts / dur / 1e9 / peaks["hbm_gbs"],
                         "peak_source": peak_src},
            "launch_ms": dur * 1e3, "traffic": traffic, "traffic_unit": "bytes per launch",
            "traffic_source": traffic_src,
            "passes_ms": {p: t * 1e3 for p, t in times.items()},
            "passes_tflops": {p: flops / t / 1e12 for p, t in times.items()}}


def dominant_kernel_roofline(torch, ctx, ops, cfg, Bl, engine, stream, engines=None):
    from paper_1510_06706_b200 import configs
    shapes = [s for s in configs.layer_shapes(cfg) if s[0] == "conv"]

    def macs(s):
        _, fi, fo, n, m, k, _ = s
        return fi * fo * np.prod(m) * np.prod(k)

    li = max(range(len(shapes)), key=lambda i: macs(shapes[i]))
    kind, fi, fo, n, m, k, s = shapes[li]
    if engine == "fft" or (engines and li < len(engines) and engines[li] == 1):
        return fft_cmac_roofline(torch, ctx, ops, Bl, fi, fo, n, k, s)
    rng = np.random.default_rng(0)
    x = torch.as_tensor(rng.uniform(0, 1, size=(Bl, fi) + tuple(n)).astype(np.float32), device="cuda")
    w = torch.as_tensor(rng.uniform(-0.01, 0.01, size=(fo, fi) + tuple(k)).astype(np.float32), device="cuda")
    g = torch.as_tensor(rng.uniform(-1, 1, size=(Bl, fo) + tuple(m)).astype(np.float32), device="cuda")
    eng = "direct" if engine in ("direct", "auto") else engine
    passes = {
        "fwd": lambda: ops.conv_fwd(ctx, x, w, k, s, act="relu", engine=eng),
        "dgrad": lambda: ops.conv_dgrad(ctx, g, w, k, s, engine=eng),
        "wgrad": lambda: ops.conv_wgrad(ctx, x, g, k, s, engine=eng),
    }
    flops = 2.0 * Bl * macs((kind, fi, fo, n, m, k, s))
    times = {}
    for name, fn in passes.items():
        if name == "dgrad" and fi == 1:
            continue
        fn()
        torch.cuda.synchronize()
        reps = 3
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        b.synchronize()
        times[name] = a.elapsed_time(b) / reps * 1e-3
    del x, g
    torch.cuda.empty_cache()
    dom = max(times, key=times.get)  # the pass of the largest layer that takes longest
    dur = times[dom]
    achieved = flops / dur / 1e12
    try:
        peak = tf32_peak_tflops(torch)
        src = "measured in-run: cuBLAS TF32 dense 8192^3 (MEASURED_PEAKS.json has bf16 only)"
    except Exception:
        peak, src = 1100.0, "nominal TF32 dense (fallback)"
    shape = f"conv f={fi}->{fo} n={tuple(n)} k={tuple(k)} s={tuple(s)} B={Bl}"
    traffic, traffic_src = None, None
    # DRAM bytes of this launch from the committed ncu capture of the same
    # shape (profiles/r01_traffic_*.json), when one exists
    import glob
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic_*.json"))):
        try:
            with open(f) as fh:
                cap = json.load(fh)
            if cap.get("shape") == shape and dom in cap.get("per_launch", {}):
                traffic = cap["per_launch"][dom]["dram_bytes"]
                traffic_src = os.path.relpath(f, ROOT) + " (ncu dram__bytes_read.sum + dram__bytes_write.sum)"
        except Exception:
            pass
    return {"bound": "tensor", "kernel": f"conv_{dom} " + shape[5:],
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "achieved_is": "algorithmic fp32 FLOP/s (2 f f' n'^3 k^3 per launch / CUDA-event duration); "
                           "3xTF32 issues 3 tensor MMAs per MAC, so tensor-pipe work is 3x this",
            "tensor_pipe_frac": 3 * achieved / peak,
            "peak_source": src, "launch_ms": dur * 1e3, "traffic": traffic, "traffic_unit": "bytes per launch",
            "traffic_source": traffic_src,
            "passes_tflops": {p: flops / t / 1e12 for p, t in times.items()}}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
