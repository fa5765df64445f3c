"""Parity at the benchmarked shapes: every conv layer of
c4 and c5 at the config's own batch (c5: 16 patches, c4: 8), on the engine
the benchmark runs it with (FFT for the 7^3 / 120->120 layers, tcgen05
direct otherwise) and on the direct engine, checked against the double CPU
oracle at sampled output voxels (forward, 1e-4), sampled input voxels (data
gradient, 1e-3) and sampled (o, i) kernel gradients summed over the batch
(1e-3), in the reference's max_rel_error (volume.hpp:170-176).

Inputs are generated on the device from a seeded torch generator (the
full-size tensors are GBs); only the slices the oracle needs come back.
Reference semantics: conv_fft.hpp:38-125 (FFT valid / adjoint / kernel
gradient), conv_direct.hpp:39-132, tests/oracles.hpp:155-252."""
import numpy as np
import pytest

from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

FWD_TOL = 1e-4
GRAD_TOL = 1e-3


def _layers(name):
    from paper_1510_06706_b200 import configs
    cfg = configs.CONFIGS[name]
    out = []
    for kind, fi, fo, n, m, k, s in configs.layer_shapes(cfg):
        if kind == "conv" and np.prod(k) > 1:
            out.append((name, cfg.batch, fi, fo, tuple(n), tuple(k), tuple(s)))
    return out


# c5 conv1-5 at B=16 (conv2-5 run FFT in the bench), c4 conv1-3 at B=8
SHAPES = _layers("c5") + _layers("c4")


def _data(shape, seed):
    _, B, fi, fo, n, k, s = shape
    m = tuple(n[a] - s[a] * (k[a] - 1) for a in range(3))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    x = torch.rand((B, fi) + n, device="cuda", generator=gen)
    bound = float(np.sqrt(6.0 / (fi * np.prod(k) + fo * np.prod(k))))
    w = (torch.rand((fo, fi) + k, device="cuda", generator=gen) * 2 - 1) * bound
    bias = (torch.rand(fo, device="cuda", generator=gen) * 2 - 1) * 0.05
    g = (torch.rand((B, fo) + m, device="cuda", generator=gen) * 2 - 1) / float(np.sqrt(fo * np.prod(k)))
    return x, w, bias, g, m


def _check(shape, y, dx, dw, x, w, bias, g, m, rng):
    _, B, fi, fo, n, k, s = shape
    wh = w.cpu().numpy()
    bh = bias.cpu().numpy()
    mv, nv = int(np.prod(m)), int(np.prod(n))
    # forward: first and last patch, first / last / a random output map, ~40 voxels each
    for b in sorted({0, B - 1}):
        xb = x[b].cpu().numpy()
        yb = y[b].cpu().numpy()
        for o in sorted({0, fo - 1, int(rng.integers(fo))}):
            idx = np.unique(np.concatenate([[0, mv - 1], rng.integers(0, mv, size=40)]))
            acc = sum(O.conv_valid_at(xb[i], wh[o, i], s, idx) for i in range(fi)) + bh[o]
            err = O.max_rel_error(yb[o].reshape(-1)[idx], np.maximum(acc, 0.0))
            assert err < FWD_TOL, ("fwd", b, o, err)
    # data gradient: sampled input voxels of two maps of two patches
    if dx is not None:
        for b in sorted({0, B - 1}):
            gb = g[b].cpu().numpy()
            dxb = dx[b].cpu().numpy()
            for i in sorted({0, fi - 1}):
                idx = np.unique(np.concatenate([[0, nv - 1], rng.integers(0, nv, size=40)]))
                ref = sum(O.conv_full_at(gb[o], O.reflect(wh[o, i]), s, idx) for o in range(fo))
                err = O.max_rel_error(dxb[i].reshape(-1)[idx], ref)
                assert err < GRAD_TOL, ("dgrad", b, i, err)
    # kernel gradient summed over the whole batch: three (o, i) edges
    dwh = dw.cpu().numpy()
    for o, i in sorted({(0, 0), (fo - 1, fi - 1), (int(rng.integers(fo)), int(rng.integers(fi)))}):
        xi = x[:, i].cpu().numpy()
        go = g[:, o].cpu().numpy()
        ref = sum(O.kernel_grad(xi[b], go[b], k, s) for b in range(B))
        err = O.max_rel_error(dwh[o, i], ref)
        assert err < GRAD_TOL, ("wgrad", o, i, err)


def _engines_for(shape):
    name, B, fi, fo, n, k, s = shape
    from paper_1510_06706_b200 import FftPlan  # noqa: F401
    out = ["direct"]
    if fi > 1 or name == "c4":  # the FFT layers of the bench (and c4 conv1, which the autotuner times)
        out.append("fft")
    return out


@pytest.mark.parametrize("engine", ["fft", "direct", "fft-dilated"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda t: f"{t[0]}-f{t[2]}x{t[3]}-n{t[4][0]}-k{t[5][0]}-s{t[6][0]}-B{t[1]}")
def test_conv_layer_full_size(ctx, shape, engine, monkeypatch):
    """engine "fft": dilated layers run the polyphase plan (phases at the
    undilated kernel's pad); "fft-dilated" (ZNN_FFT_POLY=0): the dilated
    kernel at the full pad, checked on the c4 dilated layers."""
    from paper_1510_06706_b200 import FftPlan, ops
    if engine not in _engines_for(shape) + (["fft-dilated"] if shape[0] == "c4" and max(shape[6]) > 1 else []):
        pytest.skip("layer runs direct only (1 -> f' input layer of c5), or no dilated-kernel variant")
    if engine == "fft-dilated":
        monkeypatch.setenv("ZNN_FFT_POLY", "0")
        engine = "fft"
    name, B, fi, fo, n, k, s = shape
    rng = np.random.default_rng(abs(hash(shape)) % 2**32)
    x, w, bias, g, m = _data(shape, seed=len(n) * 1000 + fi + fo + n[0])
    if engine == "fft":
        plan = FftPlan(ctx, B, fi, fo, n, k, s)
        y = plan.forward(x, w, bias=bias, act="relu")
        dx, dw = plan.backward(g, w, want_dx=fi > 1)
        plan.close()
    else:
        y = ops.conv_fwd(ctx, x, w, k, s, bias=bias, act="relu", engine="direct")
        dx = ops.conv_dgrad(ctx, g, w, k, s, engine="direct") if fi > 1 else None
        dw = ops.conv_wgrad(ctx, x, g, k, s, engine="direct")
    torch.cuda.synchronize()
    try:
        _check(shape, y, dx, dw, x, w, bias, g, m, rng)
    finally:
        del x, w, bias, g, y, dx, dw
        torch.cuda.empty_cache()


def test_fft_cmac_large_bin_grid(ctx):
    """Pads 128^3 (1,064,960 bins = 66,560 bin blocks, more than the 65,535
    grid.y limit the round-1 CMAC launches had): forward and backward run and
    match the oracle."""
    from paper_1510_06706_b200 import FftPlan
    B, fi, fo, n, k, s = 1, 2, 2, (100, 100, 100), (3, 3, 3), (1, 1, 1)
    plan = FftPlan(ctx, B, fi, fo, n, k, s)
    assert plan.info()["bins"] == 128 * 128 * 65
    shape = ("big", B, fi, fo, n, k, s)
    x, w, bias, g, m = _data(shape, seed=5)
    y = plan.forward(x, w, bias=bias, act="relu")
    dx, dw = plan.backward(g, w)
    torch.cuda.synchronize()
    _check(shape, y, dx, dw, x, w, bias, g, m, np.random.default_rng(0))
    plan.close()


def _c5_step(ctx, engines, steps=2):
    """`steps` training steps of full-size c5 (B = 16) with fixed engines:
    loss of the last step, gradients, updated parameters."""
    from paper_1510_06706_b200 import Net, configs
    cfg = configs.CONFIGS["c5"]
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    x = torch.rand((cfg.batch, cfg.in_maps) + tuple(cfg.in_dims), device="cuda", generator=gen)
    lab = (torch.rand((cfg.batch, cfg.layers[-1].width) + tuple(cfg.out_dims), device="cuda", generator=gen) < 0.5).float()
    net = Net(ctx, cfg.netspec(), cfg.out_dims, batch=cfg.batch, lr=cfg.lr, momentum=cfg.momentum, loss=cfg.loss)
    for i, e in enumerate(engines):
        net.set_layer_engine(i, e)
    net.set_params(configs.init_params(cfg, 3))
    for _ in range(steps - 1):
        net.forward_backward(x, lab, sync_loss=False)
        net.apply_update()
    loss = net.forward_backward(x, lab)
    grads = net.get_gradients()
    desc = net.describe()
    net.close()
    del x, lab
    torch.cuda.empty_cache()
    return loss, grads, desc


def test_c5_phase_major_step_equals_natural_order(ctx, monkeypatch):
    """The benchmarked c5 step keeps the groups filter -> conv3 -> conv4 -> conv5
    phase-major (executor::plan_layouts). At full size (B = 16, 120 maps) two
    steps with the bench's engines give the same loss and gradients as the
    natural-order run, whose FFT layers the tests above check against the
    oracle shape by shape; the per-layer arithmetic is identical (the same
    transforms over the same phase images), so the tolerance is 1e-5."""
    engines = ["direct", "fft", "fft", "fft", "fft", "simt"]
    loss_pm, g_pm, desc = _c5_step(ctx, engines)
    assert "phase-major groups:" in desc and len(desc.split("phase-major groups:")[-1].split("\n")[0].split()) == 3, desc
    monkeypatch.setenv("ZNN_PHASE_MAJOR", "0")
    loss_nat, g_nat, desc0 = _c5_step(ctx, engines)
    assert "phase-major groups:" not in desc0
    assert np.isfinite(loss_pm) and abs(loss_pm - loss_nat) / (abs(loss_nat) + 1) < 1e-6
    assert O.max_rel_error(g_pm, g_nat) < 1e-5
