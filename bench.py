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
    p.add_argument("--layer-engines", default=None,
                   help="comma list (direct|fft|simt per conv layer) instead of the autotuner: "
                        "ncu captures of the step without the tuner's candidate launches")
    p.add_argument("--e2e-steps", type=int, default=None)
    p.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                   help="N > 1: strong = the config's batch sharded over the ranks (default; the SGD trajectory "
                        "of the 1-GPU run), weak = every rank takes the config's whole batch (global batch x N)")
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
def cpu_baseline(cfg, warmup=1, rounds=1, budget_s=None):
    sys.path.insert(0, ROOT)
    from oracle import cpu_bench
    if budget_s is None:
        budget_s = float(os.environ.get("ZNN_CPU_BUDGET_S", "900"))
    return cpu_bench.run(cfg, warmup=warmup, rounds=rounds, mode="auto", budget_s=budget_s)


def run_reference(args):
    """The reference's own CPU implementation (engine<float>, compiled from
    /root/reference into oracle/_ref; the oracle port only if that binary is
    missing) on the same config, all host threads. One step = one reference
    round = one patch through fwd + bwd + update (engine.hpp:198-254 runs one
    sample per round): W warm-up rounds, then K measured rounds with wall time
    around each (stopping early, and saying so in "steps", only if the
    ZNN_REF_BUDGET_S budget would be exceeded)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_1510_06706_b200 import configs
    cfg = configs.CONFIGS[args.config]
    out_vox = int(np.prod(cfg.out_dims))
    # A c5 reference round takes ~55 s on 16 host threads, so the run is bounded
    # to a few minutes: at most ZNN_REF_WARMUP_MAX (1) warm-up rounds (pools and
    # plans are built in the first one) and measured rounds until the
    # ZNN_REF_BUDGET_S (240 s) budget, at least one; "steps" says how many ran.
    warm = min(args.warmup, int(os.environ.get("ZNN_REF_WARMUP_MAX", "1")))
    cb = cpu_baseline(cfg, warmup=warm, rounds=args.steps,
                      budget_s=float(os.environ.get("ZNN_REF_BUDGET_S", "240")))
    v = cb["value"]
    steps = int(cb.get("rounds", args.steps))
    line = {"metric": "train_output_voxels_per_s", "value": v, "unit": "voxels/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": int(cb.get("warmup_rounds", args.warmup)),
            "ms_per_step": out_vox / v * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": cb.get("dtype", "f32"),
            "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg.name, "global_batch": cfg.batch, "patches_per_step": 1,
                       "in_dims": cfg.in_dims, "out_dims": cfg.out_dims, "parallelism": "cpu threads",
                       "step": "one reference round = one patch (fwd + bwd + update); voxels/s is per output "
                               "voxel, so it compares directly with the GPU arm's 16-patch steps"},
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

    from paper_1510_06706_b200 import Comm, Context, Loader, Net, comm_unique_id, configs, mem_stats
    from paper_1510_06706_b200.api import profile_enable, profile_report
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
    fixed = args.layer_engines.split(",") if args.layer_engines else None
    if fixed:
        engine = "direct"
    B = cfg.batch
    if args.scaling == "weak" and world > 1:  # per-rank work fixed: the global batch grows with the ranks
        Bl, B = cfg.batch, cfg.batch * world
    else:
        lo, hi = shard_range(B, world, rank)
        Bl = hi - lo
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = Context(local, stream)
    net = Net(ctx, cfg.netspec(), cfg.out_dims, batch=Bl, global_batch=B, lr=cfg.lr,
              momentum=cfg.momentum, loss=cfg.loss, engine=engine)
    net.set_params(configs.init_params(cfg, 2026))
    if fixed:
        for i, e in enumerate(fixed):
            net.set_layer_engine(i, e)
        net.engines = [{"direct": 0, "fft": 1, "simt": 3}[e] for e in fixed]
        engine = "fixed:" + args.layer_engines
    comm = None
    if world > 1:  # the library's own NCCL communicator (per-layer allreduce buckets overlap the backward)
        uid = [comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = Comm(ctx, uid[0], world, rank)

    rng = np.random.default_rng(1000 + rank)
    n_out = cfg.layers[-1].width
    x_host = torch.from_numpy(rng.uniform(0, 1, size=(Bl, cfg.in_maps) + tuple(cfg.in_dims))
                              .astype(np.float32)).pin_memory()
    y_host = torch.from_numpy((rng.uniform(size=(Bl, n_out) + tuple(cfg.out_dims)) < 0.5)
                              .astype(np.float32)).pin_memory()
    x_dev = x_host.to("cuda", non_blocking=True)
    y_dev = y_host.to("cuda", non_blocking=True)
    torch.cuda.synchronize()
    step = DataParallelStep(net, world, comm=comm)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident timed region (in-step kernel events on for the roofline) ----
    for _ in range(args.warmup):
        step(x_dev, y_dev)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    profile_report(ctx)  # drop warm-up records
    profile_enable(ctx, True)
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
    profile_enable(ctx, False)
    launches = ctx.launches() - launches0
    kprof = profile_report(ctx)
    ms_local = ev0.elapsed_time(ev1) / args.steps
    ms = max_over_ranks(ms_local)
    mem = mem_stats(ctx)

    out_vox = int(np.prod(cfg.out_dims))
    value = B * out_vox / (ms * 1e-3)

    # ---- CUDA-graph replay of the same step (single process) ----
    graph_ms = None
    if world == 1:
        net.set_graph(True)
        for _ in range(2):
            net.train_step(x_dev, y_dev, sync_loss=False)
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(3):
            net.train_step(x_dev, y_dev, sync_loss=False)
        g1.record(stream)
        torch.cuda.synchronize()
        graph_ms = g0.elapsed_time(g1) / 3
        net.set_graph(False)

    # ---- end-to-end through the C-ABI from pinned HOST memory: every step's
    # inputs/labels copied H2D (the data provider's copy stream, overlapped
    # with the previous step) and the loss read back D2H ----
    e2e_steps = args.e2e_steps or max(2, args.steps // 2)
    h2d = (x_host.numel() + y_host.numel()) * 4
    d2h = 8
    loader = Loader(net, inputs=x_host, labels=y_host) if world == 1 else None
    if loader is not None:
        net.step_loader(loader)  # first batch's staging
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        if loader is not None:
            net.step_loader(loader)  # H2D (async, double-buffered), fwd, bwd, update, loss D2H
        else:
            x_dev.copy_(x_host, non_blocking=True)
            y_dev.copy_(y_host, non_blocking=True)
            step(x_dev, y_dev, sync_loss=True)
    e1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    e2e_ms = max_over_ranks(max(e0.elapsed_time(e1), wall * 1e3) / e2e_steps)
    e2e_value = B * out_vox / (e2e_ms * 1e-3)
    if loader is not None:
        loader.close()

    engines = list(getattr(net, "engines", []) or [])
    if rank != 0:
        if comm is not None:
            comm.close()
        if world > 1:
            dist.destroy_process_group()
        return 0

    roof, shares = roofline_from_profile(kprof, args.steps, ms_local)
    conv_tf = configs.conv_flops_per_patch(cfg) * B / (ms * 1e-3) / 1e12
    line = {
        "metric": "train_output_voxels_per_s", "value": value, "unit": "voxels/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": args.scaling if world > 1 else "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg.name, "global_batch": B, "per_gpu_batch": Bl, "in_dims": cfg.in_dims,
                   "out_dims": cfg.out_dims, "parallelism": f"dp{world}", "engine": engine,
                   "conv_engines": [{0: "direct", 1: "fft", 3: "direct-simt"}.get(e, str(e)) for e in engines]
                   if engines else None,
                   "l2": "inputs larger than L2 (per-step working set >> 126 MB)",
                   "conv_tflops_per_step_direct_equivalent": configs.conv_flops_per_patch(cfg) * B / 1e12},
        "conv_tflops_direct_equivalent": conv_tf,
        "conv_tflops_note": "effective rate: direct-convolution FLOPs (3 x 2 f f' n'^3 k^3 per conv layer) per "
                            "second of step time; the FFT layers do far fewer flops, so this exceeds the 3xTF32 "
                            "tensor ceiling and is not a hardware utilisation",
        "e2e": {"value": e2e_value, "unit": "voxels/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms, "path": "znn_net_step_loader (pinned host samples, double-buffered H2D)"
                if world == 1 else "host copy + znn_net_train_step_dp"},
        "gpu_launches": int(launches),
        "graph_ms_per_step": graph_ms,
        "memory": {"free_gb_after_step": mem["free"] / 2**30, "library_alloc_gb": mem["alloc_bytes"] / 2**30},
        "clocks": clocks.summary(),
        "roofline": roof,
        "kernel_shares": shares,
    }
    net.close()
    if not args.no_cpu_baseline and world == 1:
        try:  # 1 warm-up + 1 measured real round of the reference engine (bounded: ~2 rounds)
            line["cpu_baseline"] = cpu_baseline(cfg, warmup=1, rounds=1)
        except Exception as e:  # the baseline is reported, never the product path
            line["cpu_baseline"] = {"error": str(e)[:200]}
    print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


FP32_NOMINAL_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 148 SMs x 128 FP32 lanes x FMA x 1965 MHz = 74.4


def roofline_from_profile(kprof, steps, step_ms):
    """Roofline of the dominant kernel from the in-step CUDA events of the
    timed region: achieved = algorithmic bytes (or flops) per launch / the
    average launch duration, against MEASURED_PEAKS' HBM copy bandwidth (FFT
    passes, CMACs, max-filter) or the in-run cuBLAS TF32 rate (tcgen05
    direct convolution, 3 MMAs per fp32 MAC)."""
    peaks, peak_src = measured_peaks()
    hbm = float(peaks["hbm_gbs"])
    shares = []
    for e in sorted(kprof, key=lambda e: -e["ms"]):
        per = e["ms"] / e["launches"]
        shares.append({"kernel": e["kernel"], "launches_per_step": e["launches"] / steps,
                       "ms_per_step": e["ms"] / steps, "share_of_step": e["ms"] / steps / step_ms,
                       "gbs": e["bytes"] / e["launches"] / (per * 1e-3) / 1e9,
                       "tflops": e["flops"] / e["launches"] / (per * 1e-3) / 1e12 if e["flops"] else None})
    if not shares:
        return None, shares
    dom = shares[0]
    e = next(x for x in kprof if x["kernel"] == dom["kernel"])
    per_s = e["ms"] / e["launches"] * 1e-3
    if dom["kernel"].startswith("conv_") and "_tc" in dom["kernel"]:
        import torch
        try:
            peak, src = tf32_peak_tflops(torch), "measured in-run: cuBLAS TF32 dense 8192^3"
        except Exception:
            peak, src = 1100.0, "nominal TF32 dense (fallback)"
        ach = e["flops"] / e["launches"] / per_s / 1e12
        roof = {"bound": "tensor", "kernel": dom["kernel"], "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                "frac": ach / peak, "tensor_pipe_frac": 3 * ach / peak, "peak_source": src,
                "achieved_is": "algorithmic fp32 FLOP/s per launch; 3xTF32 issues 3 MMAs per MAC"}
    else:
        ach = e["bytes"] / e["launches"] / per_s / 1e9
        roof = {"bound": "hbm", "kernel": dom["kernel"], "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm, "peak_source": peak_src + " hbm_gbs (copy bandwidth, burst)",
                "achieved_is": "algorithmic bytes per launch (DESIGN.md 4.3b) / average in-step launch "
                               "duration (CUDA events on the executor stream over the timed region)"}
        if e["flops"]:
            tf = e["flops"] / e["launches"] / per_s / 1e12
            roof["fp32_view"] = {"achieved_tflops": tf, "peak_tflops": FP32_NOMINAL_TFLOPS,
                                 "frac": tf / FP32_NOMINAL_TFLOPS,
                                 "peak_source": "nominal FP32 FFMA rate (148 SMs x 128 lanes x 2 x 1965 MHz)"}
    roof["launch_ms"] = per_s * 1e3
    roof["algorithmic_bytes_per_launch"] = e["bytes"] / e["launches"]
    roof["traffic"], roof["traffic_source"] = committed_traffic(dom["kernel"])
    return roof, shares[:48]


def committed_traffic(kernel):
    """DRAM bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)
    from the committed --set full capture of the same kernel label, if any."""
    import glob
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic_*.json")), reverse=True):
        try:
            with open(f) as fh:
                cap = json.load(fh)
            if kernel in cap.get("per_kernel", {}):
                return cap["per_kernel"][kernel]["dram_bytes"], os.path.relpath(f, ROOT) + \
                    " (ncu dram__bytes_read.sum + dram__bytes_write.sum)"
        except Exception:
            pass
    return None, None


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
