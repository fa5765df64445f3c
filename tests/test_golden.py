"""Pin the CPU oracle to committed golden vectors produced by the reference
itself (tests/golden/make_golden.py runs oracle/_ref/znn_ref, the reference's
own code compiled unmodified). Unlike tests/test_ref_pin.py this needs neither
/root/reference nor oracle/_ref, so the pin also holds on the GPU box."""
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("name", ["tiny", "c1"])
def test_training_round_matches_golden(name):
    """oracle.train_step (B = 1, momentum 0, half-L2) == the reference's net_train_round."""
    z = np.load(os.path.join(GOLD, f"round_{name}.npz"))
    spec, od = str(z["spec"]), tuple(int(v) for v in z["out_dims"])
    g = O.parse_netspec(spec, od)
    params = z["params"]
    x = z["x"]
    flat = z["labels"]
    labels, off = [], 0
    for v in g.outputs():
        n = int(np.prod(g.nodes[v].dims))
        labels.append(flat[off:off + n].reshape(g.nodes[v].dims))
        off += n
    ol, _, op, _ = O.train_step(g, params, np.zeros(params.size), [[x]], [labels], lr=float(z["eta"]), momentum=0.0,
                                loss="l2")
    assert abs(ol - float(z["loss"])) <= 1e-10 * (1 + abs(float(z["loss"])))
    assert np.max(np.abs(op - z["new_params"])) < 1e-10


def test_maxfilter_values_and_masks_match_golden():
    """Values and argmax masks bit-exact, ties included (integer-valued inputs)."""
    z = np.load(os.path.join(GOLD, "maxfilter.npz"))
    for i in range(int(z["count"])):
        n, k, s = (tuple(int(v) for v in z[f"{key}{i}"]) for key in ("n", "k", "s"))
        out, rec = O.maxfilter_fwd(z[f"x{i}"].reshape(n), k, s)
        assert np.array_equal(out.reshape(-1), z[f"y{i}"])
        assert np.array_equal(rec.reshape(-1), z[f"mask{i}"])


def test_conv_matches_golden():
    z = np.load(os.path.join(GOLD, "conv.npz"))
    for i in range(int(z["count"])):
        n, k, s = (tuple(int(v) for v in z[f"{key}{i}"]) for key in ("n", "k", "s"))
        y = O.conv_valid(z[f"x{i}"].reshape(n), z[f"w{i}"].reshape(k), s)
        assert np.max(np.abs(y.reshape(-1) - z[f"y{i}"])) < 1e-12
