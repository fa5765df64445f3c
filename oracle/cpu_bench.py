"""CPU baseline timing — TEST/BENCH INFRASTRUCTURE ONLY.

Preferred: the reference's own task-parallel engine (engine<float>,
engine.hpp:65-254) compiled from /root/reference by oracle/ref/build.sh into
oracle/_ref/znn_ref (kind "reference"), real rounds timed on all host
threads (no extrapolation).
Fallback: the plain-C double oracle (kind "port", 1 core), timed on a
bounded per-edge sample of every conv layer and extrapolated by edge count.
"""
from __future__ import annotations

import json
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_BIN = os.path.join(_HERE, "_ref", "znn_ref")


def physical_cores():
    """acceptance.cpp:76-88 style: distinct (physical id, core id) pairs."""
    try:
        pairs, phys, core = set(), None, None
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("physical id"):
                    phys = line.split(":")[1].strip()
                elif line.startswith("core id"):
                    core = line.split(":")[1].strip()
                    pairs.add((phys, core))
        if pairs:
            return len(pairs)
    except OSError:
        pass
    return os.cpu_count() or 1


def threads():
    """All host threads the reference engine can use (its worker pool)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run(cfg, warmup=1, rounds=1, mode=None, budget_s=3000.0, port_budget_s=20.0):
    """Real rounds of the reference engine when oracle/_ref/znn_ref is built,
    else the oracle port on a bounded per-edge sample."""
    if os.path.exists(REF_BIN):
        return run_reference_engine(cfg, warmup, rounds, mode or "auto", budget_s)
    return run_port(cfg, port_budget_s)


def run_reference_engine(cfg, warmup, rounds, mode="auto", budget_s=3000.0):
    """engine<float>::run (engine.hpp:198-254) compiled from /root/reference:
    `warmup` rounds, then up to `rounds` measured rounds (one patch each, the
    reference's unit of work) with wall time around each; mode "auto" runs the
    reference's own autotune_modes first (its default policy, trainer.hpp:41)."""
    nthr = threads()
    spec_path = os.path.join("/tmp", f"znn_ref_{cfg.name}_{os.getpid()}.spec")
    with open(spec_path, "w") as f:
        f.write(cfg.netspec())
    od = ",".join(str(v) for v in cfg.out_dims)
    cmd = [REF_BIN, "bench", spec_path, od, str(nthr), str(int(warmup)), str(int(rounds)), mode, str(budget_s)]
    t0 = time.perf_counter()
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=budget_s * 3 + 600)
    wall = time.perf_counter() - t0
    os.unlink(spec_path)
    if out.returncode != 0:
        raise RuntimeError(f"reference engine failed: {out.stderr[-400:]}")
    res = json.loads(out.stdout.strip().splitlines()[-1])
    out_vox = int(np.prod(cfg.out_dims))
    value = out_vox * res["rounds"] / res["seconds"]
    return {"value": value, "unit": "voxels/s", "cores": nthr, "physical_cores": physical_cores(),
            "kind": "reference", "dtype": "f32", "mode": res["mode"], "rounds": res["rounds"],
            "warmup_rounds": res["warmup"], "seconds": res["seconds"], "warmup_seconds": res["warmup_seconds"],
            "autotune_seconds": res.get("autotune_seconds", 0.0), "round_seconds": res.get("round_seconds"),
            "process_wall_s": wall,
            "sample": f"{res['rounds']} measured round(s) of the reference engine<float> (compiled from "
                      f"/root/reference by oracle/ref/build.sh) on {cfg.name} at full size, one patch per round "
                      f"(the reference's unit of work), after {res['warmup']} warm-up round(s); conv mode "
                      f"{res['mode']}; {nthr} worker threads; wall time around each measured round"}


def run_port(cfg, budget_s):
    from . import oracle as O
    from paper_1510_06706_b200 import configs

    shapes = configs.layer_shapes(cfg)
    rng = np.random.default_rng(0)
    per_layer_budget = budget_s / max(1, len(shapes))
    total = 0.0
    sampled = []
    for kind, fi, fo, n, m, k, s in shapes:
        x = rng.uniform(0, 1, size=n)
        if kind == "conv":
            w = rng.uniform(-0.1, 0.1, size=k)
            g = rng.uniform(-1, 1, size=m)
            t0 = time.perf_counter()
            done = 0
            while done < fi * fo:
                O.conv_valid(x, w, s)
                O.conv_full(g, O.reflect(w), s)
                O.kernel_grad(x, g, k, s)
                done += 1
                if time.perf_counter() - t0 > per_layer_budget:
                    break
            per_edge = (time.perf_counter() - t0) / done
            total += per_edge * fi * fo
            sampled.append(f"{kind} {done}/{fi * fo} edges")
        else:
            t0 = time.perf_counter()
            if kind == "filter":
                y, r = O.maxfilter_fwd(x, k, s)
                O.maxfilter_bwd(y, r, n)
            else:
                y, r = O.maxpool_fwd(x, k)
                O.maxpool_bwd(y, r, k)
            total += (time.perf_counter() - t0) * fi
            sampled.append(f"{kind} 1/{fi} maps")
    out_vox = int(np.prod(cfg.out_dims))
    return {"value": out_vox / total, "unit": "voxels/s", "cores": 1, "kind": "port", "dtype": "f64",
            "sample": f"scalar double oracle, one patch of {cfg.name}: per-edge fwd+bwd+upd timed on "
                      f"[{'; '.join(sampled)}], extrapolated by edge count"}
