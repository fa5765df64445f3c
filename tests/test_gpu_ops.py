"""Op-level parity: CUDA kernels (through the C-ABI) vs the double-precision
CPU oracle on the same seeded inputs. Tolerances (BASELINE.json north_star,
measured with the reference's max_rel_error = max|a-b|/(|b|+1),
volume.hpp:170-176): forward 1e-4, gradients 1e-3; argmax masks bit-exact."""
import numpy as np
import pytest

from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FWD_TOL = 1e-4
GRAD_TOL = 1e-3
ENGINES = ["direct", "simt"]


def cuda(a, dtype=None):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda", dtype=dtype or torch.float32)


def glorot(f_in, f_out, k, rng):
    kv = int(np.prod(k))
    b = np.sqrt(6.0 / (f_in * kv + f_out * kv))
    return rng.uniform(-b, b, size=(f_out, f_in) + tuple(k)).astype(np.float32)


# (B, f_in, f_out, n, k, s): small exhaustive-ish cases + every conv layer shape of the configs
SMALL = [
    (1, 1, 1, (3, 3, 3), (2, 2, 2), (1, 1, 1)),
    (2, 3, 5, (7, 6, 9), (3, 2, 3), (1, 2, 1)),
    (1, 4, 3, (9, 9, 9), (3, 3, 3), (2, 2, 2)),
    (2, 8, 8, (20, 20, 20), (3, 3, 3), (1, 1, 1)),
    (1, 5, 7, (1, 17, 19), (1, 5, 5), (1, 2, 2)),
    (3, 2, 130, (6, 7, 8), (1, 1, 1), (1, 1, 1)),
    (1, 130, 3, (5, 5, 5), (2, 2, 2), (1, 1, 1)),
    (1, 17, 33, (13, 11, 15), (2, 3, 2), (3, 1, 2)),
]


def config_conv_shapes(batch=1):
    from paper_1510_06706_b200 import configs
    out = []
    for name in ("c1", "c2", "c3", "c4", "c5"):
        for kind, fi, fo, n, m, k, s in configs.layer_shapes(configs.CONFIGS[name]):
            if kind == "conv":
                out.append((batch, fi, fo, n, k, s))
    return out


def full_ok(shape):
    B, fi, fo, n, k, s = shape
    m = [n[a] - s[a] * (k[a] - 1) for a in range(3)]
    return fi * fo * np.prod(m) * np.prod(k) * B < 3e8


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("shape", SMALL, ids=str)
def test_conv_fwd_small(ctx, shape, engine):
    from paper_1510_06706_b200 import ops
    B, fi, fo, n, k, s = shape
    rng = np.random.default_rng(hash(shape) % 2**32)
    x = rng.uniform(0, 1, size=(B, fi) + n).astype(np.float32)
    w = glorot(fi, fo, k, rng)
    bias = rng.uniform(-0.1, 0.1, size=fo).astype(np.float32)
    for act in ("none", "relu", "logistic"):
        y = ops.conv_fwd(ctx, cuda(x), cuda(w), k, s, bias=cuda(bias), act=act, engine=engine).cpu().numpy()
        for b in range(B):
            for o in range(fo):
                acc = sum(O.conv_valid(x[b, i], w[o, i], s) for i in range(fi)) + bias[o]
                ref = O.transfer_fwd(acc, O._FN[act], 0.0) if act != "none" else acc
                assert O.max_rel_error(y[b, o], ref) < FWD_TOL, (b, o, act)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("shape", SMALL, ids=str)
def test_conv_dgrad_wgrad_small(ctx, shape, engine):
    from paper_1510_06706_b200 import ops
    B, fi, fo, n, k, s = shape
    rng = np.random.default_rng(7 + hash(shape) % 2**31)
    x = rng.uniform(0, 1, size=(B, fi) + n).astype(np.float32)
    w = glorot(fi, fo, k, rng)
    m = tuple(n[a] - s[a] * (k[a] - 1) for a in range(3))
    g = rng.uniform(-1, 1, size=(B, fo) + m).astype(np.float32)
    dx = ops.conv_dgrad(ctx, cuda(g), cuda(w), k, s, engine=engine).cpu().numpy()
    dw = ops.conv_wgrad(ctx, cuda(x), cuda(g), k, s, scale=0.5, engine=engine).cpu().numpy()
    for b in range(B):
        for i in range(fi):
            ref = sum(O.conv_full(g[b, o], O.reflect(w[o, i]), s) for o in range(fo))
            assert O.max_rel_error(dx[b, i], ref) < GRAD_TOL
    for o in range(fo):
        for i in range(fi):
            ref = 0.5 * sum(O.kernel_grad(x[b, i], g[b, o], k, s) for b in range(B))
            assert O.max_rel_error(dw[o, i], ref) < GRAD_TOL


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("shape", config_conv_shapes(), ids=str)
def test_conv_config_layers_sampled(ctx, shape, engine):
    """Every conv layer shape of configs c1..c5 at full size (B=1), checked at
    sampled output voxels / maps / taps against the double oracle."""
    from paper_1510_06706_b200 import ops
    B, fi, fo, n, k, s = shape
    if engine == "simt" and not full_ok(shape):
        pytest.skip("SIMT reference engine exercised on the small layers only")
    rng = np.random.default_rng(11)
    x = rng.uniform(0, 1, size=(B, fi) + n).astype(np.float32)
    w = glorot(fi, fo, k, rng)
    bias = rng.uniform(-0.05, 0.05, size=fo).astype(np.float32)
    m = tuple(n[a] - s[a] * (k[a] - 1) for a in range(3))
    y = ops.conv_fwd(ctx, cuda(x), cuda(w), k, s, bias=cuda(bias), act="relu", engine=engine).cpu().numpy()
    mv = int(np.prod(m))
    for o in sorted(set([0, fo - 1, int(rng.integers(fo))])):
        idx = np.unique(np.concatenate([[0, mv - 1], rng.integers(0, mv, size=40)]))
        acc = sum(O.conv_valid_at(x[0, i], w[o, i], s, idx) for i in range(fi)) + bias[o]
        ref = np.maximum(acc, 0.0)
        assert O.max_rel_error(y[0, o].reshape(-1)[idx], ref) < FWD_TOL
    g = rng.uniform(-1, 1, size=(B, fo) + m).astype(np.float32) / np.sqrt(fo * np.prod(k))
    dw = ops.conv_wgrad(ctx, cuda(x), cuda(g), k, s, engine=engine).cpu().numpy()
    pairs = {(0, 0), (fo - 1, fi - 1), (int(rng.integers(fo)), int(rng.integers(fi)))}
    for o, i in pairs:
        ref = O.kernel_grad(x[0, i], g[0, o], k, s)
        assert O.max_rel_error(dw[o, i], ref) < GRAD_TOL
    if fi > 1:
        dx = ops.conv_dgrad(ctx, cuda(g), cuda(w), k, s, engine=engine).cpu().numpy()
        nv = int(np.prod(n))
        for i in sorted(set([0, fi - 1])):
            idx = np.unique(np.concatenate([[0, nv - 1], rng.integers(0, nv, size=40)]))
            ref = sum(O.conv_full_at(g[0, o], O.reflect(w[o, i]), s, idx) for o in range(fo))
            assert O.max_rel_error(dx[0, i].reshape(-1)[idx], ref) < GRAD_TOL


FILTERS = [((6, 6, 6), (2, 2, 2), (1, 1, 1)), ((6, 6, 6), (3, 3, 3), (2, 2, 2)),
           ((1, 90, 90), (1, 2, 2), (1, 1, 1)), ((1, 81, 81), (1, 2, 2), (1, 2, 2)),
           ((31, 29, 33), (2, 2, 2), (2, 2, 2)), ((9, 8, 7), (2, 3, 1), (1, 2, 3)),
           ((1, 1, 5), (1, 1, 2), (1, 1, 1))]


@pytest.mark.parametrize("n,k,s", FILTERS, ids=str)
def test_maxfilter_bit_exact(ctx, n, k, s):
    from paper_1510_06706_b200 import ops
    rng = np.random.default_rng(3)
    for x in (rng.uniform(0, 1, size=(3,) + n).astype(np.float32),
              rng.integers(0, 3, size=(3,) + n).astype(np.float32),  # ties everywhere
              np.maximum(rng.uniform(-1, 1, size=(3,) + n), 0).astype(np.float32)):  # relu zeros
        y, mask = ops.maxfilter_fwd(ctx, cuda(x), k, s)
        y, mask = y.cpu().numpy(), mask.cpu().numpy()
        g = rng.uniform(-1, 1, size=y.shape).astype(np.float32)
        dx = ops.maxfilter_bwd(ctx, cuda(g), cuda(mask, torch.int32), k, s).cpu().numpy()
        for mp in range(3):
            ref, rec = O.maxfilter_fwd(x[mp], k, s)
            assert np.array_equal(y[mp], ref.astype(np.float32))
            assert np.array_equal(mask[mp], rec)
            rb = O.maxfilter_bwd(g[mp], rec, n)
            assert np.allclose(dx[mp], rb, rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("n,p", [((4, 4, 4), (2, 2, 2)), ((16, 16, 16), (2, 2, 2)),
                                 ((40, 40, 40), (2, 2, 2)), ((6, 4, 9), (3, 2, 3))], ids=str)
def test_maxpool_bit_exact(ctx, n, p):
    from paper_1510_06706_b200 import ops
    rng = np.random.default_rng(5)
    for x in (rng.uniform(0, 1, size=(2,) + n).astype(np.float32),
              np.ones((2,) + n, dtype=np.float32)):
        y, mask = ops.maxpool_fwd(ctx, cuda(x), p)
        y, mask = y.cpu().numpy(), mask.cpu().numpy()
        g = rng.uniform(-1, 1, size=y.shape).astype(np.float32)
        dx = ops.maxpool_bwd(ctx, cuda(g), cuda(mask, torch.int32), p).cpu().numpy()
        for mp in range(2):
            ref, rec = O.maxpool_fwd(x[mp], p)
            assert np.array_equal(y[mp], ref.astype(np.float32))
            assert np.array_equal(mask[mp], rec)
            assert np.array_equal(dx[mp], O.maxpool_bwd(g[mp], rec, p).astype(np.float32))


def test_maxfilter_backward_example(ctx):
    """test_maxops.cpp:154-174: [3,1,4,1,5], k=2 -> backward [a,0,b+c,0,d]."""
    from paper_1510_06706_b200 import ops
    x = cuda(np.array([3, 1, 4, 1, 5], dtype=np.float32).reshape(1, 1, 5))
    y, mask = ops.maxfilter_fwd(ctx, x, (1, 1, 2))
    assert mask.cpu().numpy().reshape(-1).tolist() == [0, 2, 2, 4]
    dx = ops.maxfilter_bwd(ctx, cuda(np.array([1, 2, 3, 4], dtype=np.float32).reshape(1, 1, 4)), mask,
                           (1, 1, 2))
    assert dx.cpu().numpy().reshape(-1).tolist() == [1, 0, 5, 0, 4]


@pytest.mark.parametrize("kind", ["logistic", "tanh", "relu"])
def test_transfer(ctx, kind):
    from paper_1510_06706_b200 import ops
    rng = np.random.default_rng(9)
    x = rng.uniform(-3, 3, size=(2, 3, 4, 5, 6)).astype(np.float32)
    x[0, 0, 0, 0, :2] = 0.0  # relu'(0) = 0 at the boundary
    bias = np.array([0.0, 0.2, -0.3], dtype=np.float32)
    g = rng.uniform(-1, 1, size=x.shape).astype(np.float32)
    kk = O._FN[kind]
    y = ops.transfer_fwd(ctx, cuda(x), [kind] * 3, cuda(bias)).cpu().numpy()
    gx, db = ops.transfer_bwd(ctx, cuda(g), cuda(x), [kind] * 3, cuda(bias))
    gx2, db2 = ops.transfer_bwd(ctx, cuda(g), cuda(y), [kind] * 3, cuda(bias), from_output=True)
    for f in range(3):
        ref = O.transfer_fwd(x[:, f], kk, bias[f])
        assert O.max_rel_error(y[:, f], ref) < 1e-6
        rg = O.transfer_bwd(g[:, f], x[:, f], kk, bias[f])
        assert O.max_rel_error(gx.cpu().numpy()[:, f], rg) < 1e-5
        assert O.max_rel_error(gx2.cpu().numpy()[:, f], rg) < 1e-5
        rb = O.transfer_bias_grad(x[:, f], g[:, f], kk, bias[f])
        assert abs(db.cpu().numpy()[f] - rb) / (abs(rb) + 1) < 1e-5
        assert abs(db2.cpu().numpy()[f] - rb) / (abs(rb) + 1) < 1e-5


@pytest.mark.parametrize("kind", ["l2", "ce"])
def test_loss(ctx, kind):
    from paper_1510_06706_b200 import ops
    rng = np.random.default_rng(10)
    a = rng.uniform(0.01, 0.99, size=1000).astype(np.float32)
    d = (rng.uniform(size=1000) < 0.5).astype(np.float32)
    l, g = ops.loss(ctx, kind, cuda(a), cuda(d), scale=0.25)
    rl, rg = (O.loss_l2 if kind == "l2" else O.loss_ce)(a, d)
    assert abs(l - rl) / abs(rl) < 1e-6
    assert O.max_rel_error(g.cpu().numpy(), 0.25 * rg) < 1e-6


def test_sgd_momentum(ctx):
    from paper_1510_06706_b200 import ops
    rng = np.random.default_rng(12)
    w, v, g = (rng.uniform(-1, 1, size=777).astype(np.float32) for _ in range(3))
    tw, tv = cuda(w), cuda(v)
    ops.sgd_momentum(ctx, tw, tv, cuda(g), 0.01, 0.9)
    nv = 0.9 * v.astype(np.float64) + g
    assert np.allclose(tv.cpu().numpy(), nv, atol=1e-6)
    assert np.allclose(tw.cpu().numpy(), w - 0.01 * nv, atol=1e-6)


def test_shape_errors(ctx):
    from paper_1510_06706_b200 import ShapeError, ops
    x = cuda(np.zeros((1, 1, 3, 3, 3), dtype=np.float32))
    w = cuda(np.zeros((1, 1, 2, 2, 2), dtype=np.float32))
    with pytest.raises(ShapeError):
        ops.conv_fwd(ctx, x, w, (2, 2, 2), (3, 3, 3))  # test_conv.cpp:45-49
    with pytest.raises(ShapeError):
        ops.maxpool_fwd(ctx, cuda(np.zeros((3, 4, 4), dtype=np.float32)), (2, 2, 2))
    with pytest.raises(ShapeError):
        ops.maxfilter_fwd(ctx, cuda(np.zeros((3, 3, 3), dtype=np.float32)), (2, 2, 2), (3, 3, 3))
