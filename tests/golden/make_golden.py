"""Regenerate tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref/znn_ref:
the reference's own code, /root/reference/proj/include/znn + tests/oracles.hpp,
compiled unmodified against the repo's Eigen-subset shim by oracle/ref/).
Run in the build container (where /root/reference exists and build() made
oracle/_ref): python tests/golden/make_golden.py
The fixtures let tests/test_golden.py pin the oracle where the reference is
absent (the GPU box). Inputs are seeded; outputs are whatever the reference
computes."""
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
REF = os.path.join(ROOT, "oracle", "_ref", "znn_ref")

TINY = """
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


def run(*args):
    out = subprocess.run([REF, *map(str, args)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    return out.stdout


def v3s(t):
    return ",".join(str(int(v)) for v in t)


def main():
    from oracle import oracle as O
    from paper_1510_06706_b200 import configs as C
    assert os.path.exists(REF), "build oracle/_ref first (python -c 'import __graft_entry__ as g; g.build()')"
    with tempfile.TemporaryDirectory() as d:
        # training rounds (B = 1, momentum 0, half-L2): tiny net and c1
        for name, spec, od in (("tiny", TINY, (3, 3, 3)), ("c1", C.CONFIGS["c1"].netspec(), C.CONFIGS["c1"].out_dims)):
            g = O.parse_netspec(spec, od)
            rng = np.random.default_rng(17)
            _, n = g.param_layout()
            params = rng.uniform(-0.3, 0.3, size=n)
            x = rng.uniform(0, 1, size=g.nodes[g.inputs()[0]].dims)
            labels = [rng.uniform(0, 1, size=g.nodes[v].dims) for v in g.outputs()]
            paths = [os.path.join(d, f) for f in ("s.txt", "p.bin", "x.bin", "l.bin", "o.bin")]
            open(paths[0], "w").write(spec)
            params.tofile(paths[1])
            x.tofile(paths[2])
            np.concatenate([l.reshape(-1) for l in labels]).tofile(paths[3])
            run("round", paths[0], v3s(od), paths[1], paths[2], paths[3], 0.05, paths[4])
            out = np.fromfile(paths[4], dtype=np.float64)
            np.savez_compressed(os.path.join(HERE, f"round_{name}.npz"), spec=spec, out_dims=np.array(od),
                                params=params, x=x, labels=np.concatenate([l.reshape(-1) for l in labels]),
                                eta=0.05, loss=out[0], new_params=out[1:])
        # max-filter values and argmax masks (ties: integer-valued inputs)
        rng = np.random.default_rng(5)
        cases = []
        for trial in range(24):
            n = tuple(int(v) for v in rng.integers(2, 9, size=3))
            k = tuple(int(v) for v in rng.integers(1, 4, size=3))
            s = tuple(int(v) for v in rng.integers(1, 3, size=3))
            if any(O.eff(k, s)[a] > n[a] for a in range(3)):
                continue
            x = rng.integers(0, 3, size=n).astype(np.float64) if trial % 2 else rng.uniform(size=n)
            xp, op, rp = (os.path.join(d, f) for f in ("x", "o", "r"))
            x.tofile(xp)
            run("maxfilter", xp, v3s(n), v3s(k), v3s(s), op, rp)
            cases.append((n, k, s, x.reshape(-1), np.fromfile(op), np.fromfile(rp, dtype=np.int32)))
        np.savez_compressed(os.path.join(HERE, "maxfilter.npz"),
                            **{f"{key}{i}": val for i, c in enumerate(cases)
                               for key, val in zip(("n", "k", "s", "x", "y", "mask"),
                                                   (np.array(c[0]), np.array(c[1]), np.array(c[2]), c[3], c[4], c[5]))},
                            count=len(cases))
        # valid (dilated) convolutions
        rng = np.random.default_rng(6)
        cases = []
        while len(cases) < 8:
            n = tuple(int(v) for v in rng.integers(5, 11, size=3))
            k = tuple(int(v) for v in rng.integers(1, 4, size=3))
            s = tuple(int(v) for v in rng.integers(1, 3, size=3))
            if any(O.eff(k, s)[a] > n[a] for a in range(3)):
                continue
            x, w = rng.uniform(size=n), rng.uniform(-1, 1, size=k)
            xp, wp, op = (os.path.join(d, f) for f in ("x", "w", "o"))
            x.tofile(xp)
            w.tofile(wp)
            run("conv", xp, v3s(n), wp, v3s(k), v3s(s), op)
            cases.append((n, k, s, x.reshape(-1), w.reshape(-1), np.fromfile(op)))
        np.savez_compressed(os.path.join(HERE, "conv.npz"),
                            **{f"{key}{i}": val for i, c in enumerate(cases)
                               for key, val in zip(("n", "k", "s", "x", "w", "y"),
                                                   (np.array(c[0]), np.array(c[1]), np.array(c[2]), c[3], c[4], c[5]))},
                            count=len(cases))
    print("wrote", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))


if __name__ == "__main__":
    main()
