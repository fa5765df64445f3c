"""Parity of the kernel variants that the default shapes do not reach: the
opt-in conv paths (3D box tiles with channel-blocked tap-major K for dgrad,
CTA-pair wgrad), odd row-tile counts of the clustered wgrad (a padded dummy
tile), a long batch (split-K ranges crossing patches), and FFT pads that use
the double-buffered (96) and single-buffered (128) xy plane passes.
Same oracle and tolerances as test_gpu_ops.py."""
import os

import numpy as np
import pytest

from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FWD_TOL = 1e-4
GRAD_TOL = 1e-3


def cuda(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda", dtype=torch.float32)


class env:
    """Temporarily set an environment switch read by the C++ launchers."""

    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update({k: str(v) for k, v in self.kv.items()})

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _dgrad_ref(g, w, s, i):
    return sum(O.conv_full(g[o], O.reflect(w[o, i]), s) for o in range(w.shape[0]))


@pytest.mark.parametrize("shape", [(1, 24, 20, (20, 20, 20), (3, 3, 3), (4, 4, 4)),
                                   (2, 16, 12, (13, 11, 15), (3, 2, 3), (2, 3, 2))], ids=str)
def test_dgrad_box_tiles(ctx, shape):
    """ZNN_CONV_BOX=1: box tiles + channel-blocked tap-major K (skips halo taps on all axes)."""
    from paper_1510_06706_b200 import ops
    B, fi, fo, n, k, s = shape
    rng = np.random.default_rng(21)
    w = rng.uniform(-0.2, 0.2, size=(fo, fi) + k).astype(np.float32)
    m = tuple(n[a] - s[a] * (k[a] - 1) for a in range(3))
    g = rng.uniform(-1, 1, size=(B, fo) + m).astype(np.float32)
    with env(ZNN_CONV_BOX=1):
        dx = ops.conv_dgrad(ctx, cuda(g), cuda(w), k, s).cpu().numpy()
    for b in range(B):
        for i in sorted({0, fi // 2, fi - 1}):
            assert O.max_rel_error(dx[b, i], _dgrad_ref(g[b], w, s, i)) < GRAD_TOL


@pytest.mark.parametrize("pair", [0, 1])
@pytest.mark.parametrize("shape", [(2, 3, 24, (12, 12, 12), (5, 5, 5), (1, 1, 1)),   # 3 row tiles -> padded cluster
                                   (3, 8, 40, (9, 10, 11), (3, 3, 3), (1, 2, 1)),     # patches cross split ranges
                                   (1, 6, 64, (14, 14, 14), (3, 3, 3), (2, 2, 2))], ids=str)
def test_wgrad_clusters(ctx, shape, pair):
    """Clustered wgrad (TMA multicast) and the opt-in CTA-pair variant (ZNN_WGRAD_PAIR=1)."""
    from paper_1510_06706_b200 import ops
    B, fi, fo, n, k, s = shape
    rng = np.random.default_rng(33)
    x = rng.uniform(0, 1, size=(B, fi) + n).astype(np.float32)
    m = tuple(n[a] - s[a] * (k[a] - 1) for a in range(3))
    g = rng.uniform(-1, 1, size=(B, fo) + m).astype(np.float32)
    with env(ZNN_WGRAD_PAIR=pair, ZNN_WGRAD_SPLITS=5):
        dw = ops.conv_wgrad(ctx, cuda(x), cuda(g), k, s).cpu().numpy()
    for o in sorted({0, fo // 2, fo - 1}):
        for i in sorted({0, fi - 1}):
            ref = sum(O.kernel_grad(x[b, i], g[b, o], k, s) for b in range(B))
            assert O.max_rel_error(dw[o, i], ref) < GRAD_TOL


@pytest.mark.parametrize("shape", [(1, 2, 2, (90, 90, 8), (3, 3, 3), (1, 1, 1)),      # xy pad 96 (double-buffered)
                                   (1, 1, 2, (70, 100, 12), (7, 7, 3), (1, 1, 2))], ids=str)  # xy pad 128 (single buffer)
def test_fft_large_pads(ctx, shape):
    from paper_1510_06706_b200 import ops
    B, fi, fo, n, k, s = shape
    rng = np.random.default_rng(41)
    x = rng.uniform(0, 1, size=(B, fi) + n).astype(np.float32)
    w = rng.uniform(-0.5, 0.5, size=(fo, fi) + k).astype(np.float32)
    y = ops.conv_fwd(ctx, cuda(x), cuda(w), k, s, act="none", engine="fft").cpu().numpy()
    for o in range(fo):
        ref = sum(O.conv_valid(x[0, i], w[o, i], s) for i in range(fi))
        assert O.max_rel_error(y[0, o], ref) < FWD_TOL


@pytest.mark.parametrize("od", [(26, 25, 12), (4, 3, 65)], ids=["pads40x40x20", "pads12x12x80"])
def test_fft_radix5_pads_backward(ctx, od):
    """One SGD step of a net whose FFT layer has pads with a factor 5 (20, 40,
    80), data and weight gradients included, against the double oracle. The
    FFT layer (3 -> 2 maps, 5^3 sparsity 2) is the second conv, so its input
    gradient is needed."""
    from paper_1510_06706_b200 import Net
    spec = ("[node in] role=input\n"
            + "".join(f"[node h{i}]\n[node t{i}]\n" for i in range(3))
            + "[node o0] role=output\n[node o1] role=output\n"
            + "".join(f"[edge c{i}] from=in to=h{i} type=conv kernel=1,1,1\n" for i in range(3))
            + "".join(f"[edge t{i}] from=h{i} to=t{i} type=transfer fn=tanh\n" for i in range(3))
            + "".join(f"[edge e{i}{j}] from=t{i} to=o{j} type=conv kernel=5,5,5 sparsity=2,2,2\n"
                      for i in range(3) for j in range(2)))
    n = tuple(d + 8 for d in od)
    B = 2
    net = Net(ctx, spec, od, batch=B, loss="l2", lr=0.01)
    net.set_layer_engine(1, "fft")
    rng = np.random.default_rng(17)
    params = rng.uniform(-0.3, 0.3, size=net.num_params).astype(np.float32)
    net.set_params(params)
    x = rng.uniform(0, 1, size=(B, 1) + n).astype(np.float32)
    lab = rng.uniform(0, 1, size=(B, 2) + od).astype(np.float32)
    loss = net.forward_backward(cuda(x), cuda(lab))
    grads = net.get_gradients()
    net.apply_update()
    g = O.parse_netspec(spec, od)
    rl, rg, rp, _ = O.train_step(g, params.astype(np.float64), np.zeros(params.size),
                                 [[x[b, 0]] for b in range(B)], [[lab[b, o] for o in range(2)] for b in range(B)],
                                 0.01, 0.0, "l2")
    assert abs(loss - rl) / (abs(rl) + 1) < FWD_TOL
    assert O.max_rel_error(grads, rg) < GRAD_TOL
    assert O.max_rel_error(net.get_params(), rp) < GRAD_TOL
