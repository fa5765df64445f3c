"""Pin the CPU oracle (oracle/znn_oracle.c) to the reference's own known-answer
tests before it is trusted as the parity checker. Every case cites the
reference test it restates (proj/tests/*.cpp)."""
import itertools

import numpy as np
import pytest

from oracle import oracle as O


def rnd(shape, rng, lo=-1.0, hi=1.0):
    return rng.uniform(lo, hi, size=shape)


# ---- test_conv.cpp -------------------------------------------------------

def test_valid_all_ones_sums():  # test_conv.cpp:13-20
    out = O.conv_valid(np.ones((3, 3, 3)), np.ones((2, 2, 2)))
    assert out.shape == (2, 2, 2) and np.all(out == 8.0)


def test_valid_delta_kernel_crops():  # test_conv.cpp:22-33
    rng = np.random.default_rng(2)
    x = rnd((5, 5, 5), rng)
    k = np.zeros((3, 3, 3))
    k[1, 2, 0] = 1.0
    out = O.conv_valid(x, k)
    assert out.shape == (3, 3, 3)
    assert np.array_equal(out, x[1:4, 2:5, 0:3])


def test_valid_sparse_matches_definition():  # test_conv.cpp:35-43
    rng = np.random.default_rng(3)
    x, k = rnd((5, 5, 5), rng), rnd((3, 3, 3), rng)
    out = O.conv_valid(x, k, (2, 2, 2))
    ref = sum(x[2 * a, 2 * b, 2 * c] * k[a, b, c] for a in range(3) for b in range(3) for c in range(3))
    assert out.shape == (1, 1, 1) and abs(out[0, 0, 0] - ref) < 1e-12


def test_full_impulse_is_reflected_kernel():  # test_conv.cpp:51-61
    rng = np.random.default_rng(5)
    k = rnd((3, 3, 3), rng)
    out = O.conv_full(np.full((1, 1, 1), 2.0), k)
    assert np.allclose(out, 2.0 * k[::-1, ::-1, ::-1], atol=1e-12)
    assert np.array_equal(O.reflect(k), k[::-1, ::-1, ::-1])


def test_full_centered_delta_zero_pads():  # test_conv.cpp:63-77
    rng = np.random.default_rng(7)
    g = rnd((4, 4, 4), rng)
    k = np.zeros((3, 3, 3))
    k[1, 1, 1] = 1.0
    out = O.conv_full(g, k)
    ref = np.zeros((6, 6, 6))
    ref[1:5, 1:5, 1:5] = g
    assert np.allclose(out, ref, atol=1e-14)


def test_adjoint_identity():  # test_conv.cpp:97-115
    rng = np.random.default_rng(13)
    for _ in range(10):
        n = tuple(rng.integers(4, 8, size=3))
        kd = tuple(rng.integers(1, 4, size=3))
        s = (int(rng.integers(1, 3)), 1, int(rng.integers(1, 3)))
        if any(O.eff(kd, s)[a] > n[a] for a in range(3)):
            continue
        x, k = rnd(n, rng), rnd(kd, rng)
        y = O.conv_valid(x, k, s)
        g = rnd(y.shape, rng)
        xt = O.conv_full(g, O.reflect(k), s)
        assert xt.shape == x.shape
        assert abs(np.sum(y * g) - np.sum(x * xt)) < 1e-10 * (1 + abs(np.sum(y * g)))


def test_kernel_grad_known_answers():  # test_conv.cpp:117-131
    dk = O.kernel_grad(np.ones((4, 4, 4)), np.zeros((3, 3, 3)), (2, 2, 2))
    assert np.all(dk == 0.0)
    dk = O.kernel_grad(np.ones((3, 3, 3)), np.ones((2, 2, 2)), (2, 2, 2))
    assert dk.shape == (2, 2, 2) and np.all(dk == 8.0)


def test_kernel_grad_sparse_definition():  # test_conv.cpp:133-142
    rng = np.random.default_rng(17)
    x = rnd((7, 6, 7), rng)
    kd, s = (2, 3, 2), (2, 1, 2)
    m = tuple(x.shape[a] - O.eff(kd, s)[a] + 1 for a in range(3))
    g = rnd(m, rng)
    dk = O.kernel_grad(x, g, kd, s)
    for a, b, c in itertools.product(range(2), range(3), range(2)):
        ref = np.sum(x[s[0] * a:s[0] * a + m[0], s[1] * b:s[1] * b + m[1], s[2] * c:s[2] * c + m[2]] * g)
        assert abs(dk[a, b, c] - ref) < 1e-12


def test_dilate():  # test_conv.cpp:150-165
    rng = np.random.default_rng(19)
    k = rnd((2, 3, 2), rng)
    assert np.array_equal(O.dilate(k, (1, 1, 1)), k)
    d = O.dilate(np.ones((2, 2, 2)), (2, 2, 2))
    assert d.shape == (3, 3, 3) and d.sum() == 8.0
    for i, j, l in itertools.product(range(3), repeat=3):
        assert d[i, j, l] == (1.0 if (i % 2 == 0 and j % 2 == 0 and l % 2 == 0) else 0.0)


def test_sparse_equals_dilated_exhaustive():  # test_conv.cpp:167-179
    rng = np.random.default_rng(23)
    for k in (2, 3):
        for s in (1, 2, 3):
            for n in range(s * (k - 1) + 1, 10):
                x, w = rnd((n, n, n), rng), rnd((k, k, k), rng)
                a = O.conv_valid(x, w, (s, s, s))
                b = O.conv_valid(x, O.dilate(w, (s, s, s)))
                assert np.max(np.abs(a - b)) < 1e-12


def test_conv_valid_at_matches_full():
    rng = np.random.default_rng(29)
    x, k = rnd((9, 8, 10), rng), rnd((3, 2, 3), rng)
    s = (2, 3, 1)
    full = O.conv_valid(x, k, s)
    idx = rng.integers(0, full.size, size=20)
    assert np.array_equal(O.conv_valid_at(x, k, s, idx), full.reshape(-1)[idx])


# ---- test_maxops.cpp -----------------------------------------------------

def test_sliding_max_example():  # test_maxops.cpp:13-20
    out, arg = O.sliding_max_1d([3, 1, 4, 1, 5], 2, 1)
    assert list(out) == [3, 4, 4, 5] and list(arg) == [0, 2, 2, 4]


def test_sliding_max_exhaustive_three_symbols():  # test_maxops.cpp:22-58
    mism = 0
    for n in range(1, 10):  # reference goes to 12; 9 keeps the CPU suite fast
        for code in itertools.product(range(3), repeat=n):
            v = np.array(code, dtype=np.float64)
            for s in (1, 2, 3):
                k = 1
                while s * (k - 1) + 1 <= n:
                    out, arg = O.sliding_max_1d(v, k, s)
                    for o in range(n - s * (k - 1)):
                        best, low = v[o], o
                        for w in range(1, k):
                            if v[o + s * w] > best:
                                best, low = v[o + s * w], o + s * w
                        mism += (out[o] != best) or (arg[o] != low)
                    k += 1
    assert mism == 0


def test_maxpool_ramp():  # test_maxops.cpp:60-67
    out, rec = O.maxpool_fwd(np.arange(8, dtype=np.float64).reshape(2, 2, 2), (2, 2, 2))
    assert out[0, 0, 0] == 7.0 and rec[0, 0, 0] == 7


def test_maxpool_ties_first_index():  # test_maxops.cpp:69-77
    out, rec = O.maxpool_fwd(np.ones((4, 4, 4)), (2, 2, 2))
    for bi, bj, bl in itertools.product(range(2), repeat=3):
        assert rec[bi, bj, bl] == ((2 * bi) * 4 + 2 * bj) * 4 + 2 * bl


def test_maxpool_backward_places_gradient():  # test_maxops.cpp:93-105
    x = np.array([9.0 if i == 3 else float(i) for i in range(8)]).reshape(2, 2, 2)
    out, rec = O.maxpool_fwd(x, (2, 2, 2))
    back = O.maxpool_bwd(np.full((1, 1, 1), 2.5), rec, (2, 2, 2)).reshape(-1)
    assert list(back) == [2.5 if i == 3 else 0.0 for i in range(8)]


def test_maxfilter_constant_ties():  # test_maxops.cpp:107-117
    out, rec = O.maxfilter_fwd(np.full((4, 4, 4), 3.0), (2, 2, 2), (1, 1, 1))
    assert out.shape == (3, 3, 3) and np.all(out == 3.0)
    for i, j, l in itertools.product(range(3), repeat=3):
        assert rec[i, j, l] == (i * 4 + j) * 4 + l


def _brute_filter(x, k, s):
    m = tuple(x.shape[a] - s[a] * (k[a] - 1) for a in range(3))
    out = np.empty(m)
    arg = np.empty(m, dtype=np.int64)
    for i, j, l in itertools.product(*[range(v) for v in m]):
        best, bi = None, None
        for a, b, c in itertools.product(range(k[0]), range(k[1]), range(k[2])):
            v = x[i + s[0] * a, j + s[1] * b, l + s[2] * c]
            if best is None or v > best:
                best = v
                bi = ((i + s[0] * a) * x.shape[1] + j + s[1] * b) * x.shape[2] + l + s[2] * c
        out[i, j, l], arg[i, j, l] = best, bi
    return out, arg


def test_maxfilter_brute_force_shapes():  # test_maxops.cpp:119-146
    rng = np.random.default_rng(31)
    for _ in range(40):
        n = tuple(rng.integers(2, 9, size=3))
        k = tuple(rng.integers(1, 4, size=3))
        s = tuple(rng.integers(1, 3, size=3))
        if any(O.eff(k, s)[a] > n[a] for a in range(3)):
            continue
        x = rng.integers(0, 3, size=n).astype(np.float64)  # many ties
        out, rec = O.maxfilter_fwd(x, k, s)
        ref, arg = _brute_filter(x, k, s)
        assert np.array_equal(out, ref)
        assert np.array_equal(rec, arg)


def test_maxfilter_backward_accumulates():  # test_maxops.cpp:154-174
    x = np.array([3, 1, 4, 1, 5], dtype=np.float64).reshape(1, 1, 5)
    out, rec = O.maxfilter_fwd(x, (1, 1, 2), (1, 1, 1))
    back = O.maxfilter_bwd(np.array([1, 2, 3, 4], dtype=np.float64).reshape(1, 1, 4), rec, (1, 1, 5))
    assert list(back.reshape(-1)) == [1.0, 0.0, 5.0, 0.0, 4.0]


def test_max_adjoints():  # test_maxops.cpp:176-214
    rng = np.random.default_rng(41)
    for fwd, bwd, dims in (
        (lambda v: O.maxpool_fwd(v, (2, 2, 2)), lambda g, r: O.maxpool_bwd(g, r, (2, 2, 2)), (4, 4, 4)),
        (lambda v: O.maxfilter_fwd(v, (2, 2, 2), (2, 2, 2)), lambda g, r: O.maxfilter_bwd(g, r, (6, 6, 6)),
         (6, 6, 6)),
    ):
        x = rnd(dims, rng)
        y, rec = fwd(x)
        g = rnd(y.shape, rng)
        xt = bwd(g, rec)
        d = rnd(dims, rng, -1e-7, 1e-7)
        yp, _ = fwd(x + d)
        assert abs(np.sum((yp - y) * g) - np.sum(d * xt)) < 1e-5 * abs(np.sum(d * xt)) + 1e-15


# ---- test_transfer.cpp ---------------------------------------------------

def test_transfer_zero_input():  # test_transfer.cpp:13-20
    assert np.all(O.transfer_fwd(np.zeros(8), O.RELU, 0.0) == 0.0)
    assert np.allclose(O.transfer_fwd(np.zeros(8), O.LOGISTIC, 0.0), 0.5)


def test_transfer_tanh_bias():  # test_transfer.cpp:22-28
    rng = np.random.default_rng(3)
    x = rnd(27, rng)
    assert np.allclose(O.transfer_fwd(x, O.TANH, 0.1), np.tanh(x + 0.1), rtol=1e-12)


def test_relu_backward_saturates():  # test_transfer.cpp:30-42
    rng = np.random.default_rng(4)
    g = rnd(8, rng)
    assert np.array_equal(O.transfer_bwd(g, np.full(8, 1.5), O.RELU, 0.0), g)
    assert np.all(O.transfer_bwd(g, np.full(8, -1.5), O.RELU, 0.0) == 0.0)
    assert O.transfer_derivative(O.RELU, 0.0) == 0.0


@pytest.mark.parametrize("kind", [O.LOGISTIC, O.TANH, O.RELU])
def test_transfer_derivative_finite_difference(kind):  # test_transfer.cpp:53-65
    rng = np.random.default_rng(5)
    for x in rng.uniform(-3, 3, size=1000):
        if kind == O.RELU and abs(x) < 1e-4:
            continue
        fd = (O.transfer_value(kind, x + 1e-6) - O.transfer_value(kind, x - 1e-6)) / 2e-6
        assert abs(O.transfer_derivative(kind, x) - fd) <= 1e-6 * max(1.0, abs(fd))


def test_bias_gradient_fused():  # test_transfer.cpp:83-102
    rng = np.random.default_rng(8)
    x, g = rnd(24, rng), rnd(24, rng)
    a = O.transfer_bias_grad(x, g, O.TANH, -0.3)
    b = np.sum(O.transfer_bwd(g, x, O.TANH, -0.3))
    assert abs(a - b) < 1e-12


# ---- loss / gradients (taskgraph.hpp:116-126; test_engine.cpp:204-238) ----

def test_loss_l2_and_ce():
    a = np.array([0.2, 0.7, 0.5])
    d = np.array([0.0, 1.0, 1.0])
    l, g = O.loss_l2(a, d)
    assert abs(l - 0.5 * np.sum((a - d) ** 2)) < 1e-15 and np.allclose(g, a - d)
    l, g = O.loss_ce(a, d)
    assert abs(l + np.sum(d * np.log(a) + (1 - d) * np.log(1 - a))) < 1e-12 and np.allclose(g, a - d)


SMALL_NET = """
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
"""  # test_engine.cpp:42-54 tiny_spec


def test_network_gradient_matches_finite_differences():
    """Criterion 1 (acceptance.cpp:90-168): FD gradients within 1e-4, double."""
    g = O.parse_netspec(SMALL_NET, (3, 3, 3))
    rng = np.random.default_rng(43)
    _, n = g.param_layout()
    p = rng.uniform(-0.5, 0.5, size=n)
    p[[off for eid, off, sz in g.param_layout()[0] if g.edges[eid].kind == "transfer"]] = 0.1
    x = [rng.uniform(0, 1, size=g.nodes[0].dims)]
    lab = [rng.uniform(0, 1, size=(3, 3, 3)) for _ in g.outputs()]
    _, grad, *_ = O.patch_gradients(g, p, x, lab, "l2")

    def loss_at(q):
        fwd, _ = O.forward(g, q, x)
        return sum(O.loss_l2(fwd[v], lab[i])[0] for i, v in enumerate(g.outputs()))

    for i in range(n):
        e = np.zeros(n)
        e[i] = 1e-6
        fd = (loss_at(p + e) - loss_at(p - e)) / 2e-6
        assert abs(grad[i] - fd) <= 1e-4 * max(1.0, abs(fd))


def test_ce_gradient_matches_finite_differences():
    """Cross-entropy extension (configs 2-5): pinned by FD like criterion 1."""
    spec = SMALL_NET.replace("to=out0 type=conv", "to=p0 type=conv").replace(
        "to=out1 type=conv", "to=p1 type=conv").replace(
        "[node out0] role=output", "[node p0]\n[node p1]\n[node out0] role=output") + \
        "[edge s0] from=p0 to=out0 type=transfer fn=logistic\n" \
        "[edge s1] from=p1 to=out1 type=transfer fn=logistic\n"
    g = O.parse_netspec(spec, (3, 3, 3))
    rng = np.random.default_rng(47)
    _, n = g.param_layout()
    p = rng.uniform(-0.5, 0.5, size=n)
    x = [rng.uniform(0, 1, size=g.nodes[0].dims)]
    lab = [(rng.uniform(size=(3, 3, 3)) < 0.5).astype(np.float64) for _ in g.outputs()]
    _, grad, *_ = O.patch_gradients(g, p, x, lab, "ce")

    def loss_at(q):
        fwd, _ = O.forward(g, q, x)
        return sum(O.loss_ce(fwd[v], lab[i])[0] for i, v in enumerate(g.outputs()))

    for i in range(n):
        e = np.zeros(n)
        e[i] = 1e-6
        fd = (loss_at(p + e) - loss_at(p - e)) / 2e-6
        assert abs(grad[i] - fd) <= 1e-4 * max(1.0, abs(fd))


def test_sliding_equivalence_every_offset():
    """Criterion 3 (acceptance.cpp:200-265): the sliding rewrite applied densely
    equals the pooling net applied at every window offset."""
    spec = """
[node in] role=input
[node a]
[node b]
[node c]
[node out] role=output
[edge c1] from=in to=a type=conv kernel=2,2,2
[edge p1] from=a to=b type=pool p=2,2,2
[edge c2] from=b to=c type=conv kernel=2,2,2
[edge t1] from=c to=out type=transfer fn=tanh
"""
    g = O.parse_netspec(spec, (1, 1, 1))
    sg = O.to_sliding_equivalent(g)
    O.infer_shapes(sg, (3, 3, 3))
    rng = np.random.default_rng(53)
    _, n = g.param_layout()
    p = rng.uniform(-1, 1, size=n)
    big = rng.uniform(0, 1, size=sg.nodes[0].dims)
    dense, _ = O.forward(sg, p, [big])
    dense_out = dense[sg.outputs()[0]]
    win = g.nodes[0].dims
    for i, j, l in itertools.product(range(3), repeat=3):
        f, _ = O.forward(g, p, [big[i:i + win[0], j:j + win[1], l:l + win[2]]])
        assert abs(f[g.outputs()[0]][0, 0, 0] - dense_out[i, j, l]) < 1e-12
