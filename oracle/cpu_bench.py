"""CPU baseline timing — TEST/BENCH INFRASTRUCTURE ONLY.

Preferred: the reference's own task-parallel engine (engine<float>,
engine.hpp:65-254) compiled from /root/reference by oracle/ref/build.sh into
oracle/_ref/znn_ref (kind "reference"), run on all host cores; configs whose
round exceeds the budget report the per-edge estimate (see znn_ref.cpp).
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


def run(cfg, budget_s=20.0, mode=None):
    if os.path.exists(REF_BIN):
        return run_reference_engine(cfg, budget_s, mode or ("auto" if cfg.engine == "auto" else "direct"))
    return run_port(cfg, budget_s)


def run_reference_engine(cfg, budget_s, mode="direct"):
    threads = physical_cores()
    spec_path = os.path.join("/tmp", f"znn_ref_{cfg.name}_{os.getpid()}.spec")
    with open(spec_path, "w") as f:
        f.write(cfg.netspec())
    od = ",".join(str(v) for v in cfg.out_dims)
    # predicted round time from the reference's own per-edge task bodies
    est = subprocess.run([REF_BIN, "estimate", spec_path, od, str(threads)], capture_output=True, text=True,
                         timeout=900)
    if est.returncode == 0:
        e = json.loads(est.stdout.strip().splitlines()[-1])
        if e["round_seconds"] * 2.0 > budget_s:
            os.unlink(spec_path)
            out_vox = int(np.prod(cfg.out_dims))
            return {"value": out_vox / e["round_seconds"], "unit": "voxels/s", "cores": threads,
                    "kind": "reference", "dtype": "f32", "estimated": True,
                    "sample": f"one full {cfg.name} round exceeds the {budget_s:.0f}s budget: every edge signature's "
                              f"reference task bodies (conv_valid_direct + conv_full_direct(reflect) + "
                              f"kernel_gradient_direct, transfer/filter/pool fwd+bwd; engine.hpp:582-829) timed "
                              f"single-threaded (median of 3), summed over all {cfg.name} edges and divided by "
                              f"{threads} threads (the paper's linear speedup, optimistic for the CPU)"}
    cmd = [REF_BIN, "bench", spec_path, od, str(threads), str(budget_s), mode]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=budget_s * 20 + 600)
    os.unlink(spec_path)
    if out.returncode != 0:
        raise RuntimeError(f"reference engine failed: {out.stderr[-400:]}")
    res = json.loads(out.stdout.strip().splitlines()[-1])
    out_vox = int(np.prod(cfg.out_dims))
    value = out_vox * res["rounds"] / res["seconds"]
    return {"value": value, "unit": "voxels/s", "cores": threads, "kind": "reference",
            "dtype": "f32",
            "sample": f"{res['rounds']} measured round(s) (1 patch each, after {res['warmup']} warm-up round) of "
                      f"the reference engine<float> (compiled from /root/reference, oracle/ref/build.sh) on "
                      f"{cfg.name} at full size, conv mode {res['mode']}, {threads} worker threads, wall time "
                      f"around the measured rounds"}


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
