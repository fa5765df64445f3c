"""Pin the plain-C oracle to the REFERENCE ITSELF: oracle/_ref/znn_ref is the
reference's own code (/root/reference/proj/include/znn + tests/oracles.hpp)
compiled unmodified against the repo's Eigen-subset shim (oracle/ref/).
Both sides run in double on the same seeded inputs."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "znn_ref")
pytestmark = pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built")


def run(*args):
    out = subprocess.run([REF, *map(str, args)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    return out.stdout


def v3s(t):
    return ",".join(str(int(v)) for v in t)


def ref_round(spec, out_dims, params, x, labels, eta):
    with tempfile.TemporaryDirectory() as d:
        paths = [os.path.join(d, n) for n in ("s.txt", "p.bin", "x.bin", "l.bin", "o.bin")]
        open(paths[0], "w").write(spec)
        np.asarray(params, np.float64).tofile(paths[1])
        np.asarray(x, np.float64).tofile(paths[2])
        np.concatenate([np.asarray(l, np.float64).reshape(-1) for l in labels]).tofile(paths[3])
        run("round", paths[0], v3s(out_dims), paths[1], paths[2], paths[3], eta, paths[4])
        out = np.fromfile(paths[4], dtype=np.float64)
    return out[0], out[1:]


def net_cases():
    from paper_1510_06706_b200 import configs as C
    tiny = """
[node in] role=input
[node h0]
[node h1]
[node t0]
[node t1]
[node out0] role=output
[node out1] role=output
[edge c0] from=in to=h0 type=conv kernel=2,2,2
[edge c1] from=in to=h1 type=conv kernel=2,2,2
[edge t0] from=h0 to=t0 type=transfer fn=tanh
[edge t1] from=h1 to=t1 type=transfer fn=logistic
[edge c2] from=t0 to=out0 type=conv kernel=2,2,2
[edge c3] from=t0 to=out1 type=conv kernel=2,2,2
[edge c4] from=t1 to=out0 type=conv kernel=2,2,2
[edge c5] from=t1 to=out1 type=conv kernel=2,2,2
"""  # test_engine.cpp:42-54
    cases = [("tiny", tiny, (3, 3, 3)), ("c1", C.CONFIGS["c1"].netspec(), C.CONFIGS["c1"].out_dims)]
    for name, wd, od in (("c2", 8, (1, 5, 5)), ("c3", 10, (2, 2, 2)), ("c4", 20, (1, 1, 1)), ("c5", 30, (1, 1, 1))):
        c = C.scaled(name, wd, od, batch=1)
        cases.append((c.name, c.netspec(), c.out_dims))
    return cases


@pytest.mark.parametrize("name,spec,od", net_cases(), ids=lambda v: v if isinstance(v, str) and len(v) < 20 else "")
def test_training_round_matches_reference(name, spec, od):
    """oracle.train_step (B=1, momentum 0, half-L2) == reference net_train_round."""
    g = O.parse_netspec(spec, od)
    rng = np.random.default_rng(17)
    _, n = g.param_layout()
    params = rng.uniform(-0.3, 0.3, size=n)
    x = rng.uniform(0, 1, size=g.nodes[g.inputs()[0]].dims)
    labels = [rng.uniform(0, 1, size=g.nodes[v].dims) for v in g.outputs()]
    rl, rp = ref_round(spec, od, params, x, labels, 0.05)
    ol, _, op, _ = O.train_step(g, params, np.zeros(n), [[x]], [labels], lr=0.05, momentum=0.0, loss="l2")
    assert abs(ol - rl) <= 1e-10 * (1 + abs(rl))
    assert np.max(np.abs(op - rp)) < 1e-10


def test_maxfilter_masks_match_reference():
    rng = np.random.default_rng(5)
    with tempfile.TemporaryDirectory() as d:
        for trial in range(30):
            n = tuple(int(v) for v in rng.integers(2, 10, size=3))
            k = tuple(int(v) for v in rng.integers(1, 4, size=3))
            s = tuple(int(v) for v in rng.integers(1, 3, size=3))
            if any(O.eff(k, s)[a] > n[a] for a in range(3)):
                continue
            x = rng.integers(0, 3, size=n).astype(np.float64) if trial % 2 else rng.uniform(size=n)
            xp, op, rp = (os.path.join(d, f) for f in ("x", "o", "r"))
            x.tofile(xp)
            run("maxfilter", xp, v3s(n), v3s(k), v3s(s), op, rp)
            ref_out, ref_rec = np.fromfile(op), np.fromfile(rp, dtype=np.int32)
            out, rec = O.maxfilter_fwd(x, k, s)
            assert np.array_equal(out.reshape(-1), ref_out)
            assert np.array_equal(rec.reshape(-1), ref_rec)


def test_conv_matches_reference():
    rng = np.random.default_rng(6)
    with tempfile.TemporaryDirectory() as d:
        for _ in range(10):
            n = tuple(int(v) for v in rng.integers(5, 12, size=3))
            k = tuple(int(v) for v in rng.integers(1, 4, size=3))
            s = tuple(int(v) for v in rng.integers(1, 3, size=3))
            if any(O.eff(k, s)[a] > n[a] for a in range(3)):
                continue
            x, w = rng.uniform(size=n), rng.uniform(-1, 1, size=k)
            xp, wp, op = (os.path.join(d, f) for f in ("x", "w", "o"))
            x.tofile(xp)
            w.tofile(wp)
            run("conv", xp, v3s(n), wp, v3s(k), v3s(s), op)
            assert np.max(np.abs(O.conv_valid(x, w, s).reshape(-1) - np.fromfile(op))) < 1e-12


def test_reference_engine_bench_runs():
    from paper_1510_06706_b200 import configs as C
    from oracle import cpu_bench
    res = cpu_bench.run(C.CONFIGS["c1"], budget_s=1.0)
    assert res["kind"] == "reference" and res["value"] > 0
