"""Runtime around the kernels: CUDA-graph replay of the step,
zero device allocations in the steady state (the analogue of the
reference's acceptance criterion 9, acceptance.cpp:637-656), memory
planning from cudaMemGetInfo, the data provider with pinned double-buffered
H2D (trainer.hpp:87-166) and ZNNV files (volume_io.hpp), the NCCL
data-parallel step (one rank here: only one GPU is available), and the
per-layer autotuner entry point (trainer.hpp:181-250)."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _case(name="c5", wd=24, od=(1, 1, 1), batch=2, seed=3):
    from paper_1510_06706_b200 import configs as C
    cfg = C.scaled(name, wd, od, batch=batch)
    rng = np.random.default_rng(seed)
    params = C.init_params(cfg, seed)
    x = rng.uniform(0, 1, size=(cfg.batch, cfg.in_maps) + tuple(cfg.in_dims)).astype(np.float32)
    lab = (rng.uniform(size=(cfg.batch, cfg.layers[-1].width) + tuple(cfg.out_dims)) < 0.5).astype(np.float32)
    return cfg, params, x, lab


def _net(ctx, cfg, params, fft=True):
    from paper_1510_06706_b200 import Net
    net = Net(ctx, cfg.netspec(), cfg.out_dims, batch=cfg.batch, lr=cfg.lr, momentum=cfg.momentum, loss=cfg.loss)
    if fft:
        for li, L in enumerate(cfg.conv_layers()):
            if np.prod(L.k) > 1 and li > 0:
                net.set_layer_engine(li, "fft")
    net.set_params(params)
    return net


@pytest.fixture
def stream_ctx():
    """A context on a non-default stream (graph capture needs one)."""
    from paper_1510_06706_b200 import Context
    st = torch.cuda.Stream()
    c = Context(0, st)
    yield c, st
    c.close()


def test_graph_replay_is_bit_identical_and_allocation_free(stream_ctx):
    from paper_1510_06706_b200 import mem_stats
    ctx, st = stream_ctx
    cfg, params, x, lab = _case()
    xd, ld = torch.as_tensor(x, device="cuda"), torch.as_tensor(lab, device="cuda")
    torch.cuda.synchronize()
    ref = _net(ctx, cfg, params)
    ref_losses = [ref.train_step(xd, ld) for _ in range(5)]
    ref_p = ref.get_params()
    ref.close()

    net = _net(ctx, cfg, params)
    net.set_graph(True)
    losses = [net.train_step(xd, ld)]  # eager warm-up step
    assert not net.graph_captured()
    losses.append(net.train_step(xd, ld))  # captured + replayed
    assert net.graph_captured()
    a0 = mem_stats(ctx)["allocs"]
    launches0 = ctx.launches()
    for _ in range(3):
        losses.append(net.train_step(xd, ld))
    # steps 3..5 replay the graph: no device allocation, no kernel issued from the host
    assert mem_stats(ctx)["allocs"] == a0
    assert ctx.launches() == launches0
    assert losses == ref_losses
    assert np.array_equal(net.get_params(), ref_p)


def test_eager_steady_state_allocates_nothing(ctx):
    """Without graphs too: after the first step every buffer (activations,
    spectra, kernel-spectrum pool, scratch arena) is at its final size."""
    from paper_1510_06706_b200 import mem_stats
    cfg, params, x, lab = _case("c4", 16, (2, 2, 2))
    net = _net(ctx, cfg, params)
    xd, ld = torch.as_tensor(x, device="cuda"), torch.as_tensor(lab, device="cuda")
    net.train_step(xd, ld)
    a0 = mem_stats(ctx)["allocs"]
    for _ in range(3):
        net.train_step(xd, ld)
    assert mem_stats(ctx)["allocs"] == a0


def test_pingpong_gradients_match_kept_images(ctx, monkeypatch):
    """Two ping-pong backward buffers (default) == one gradient buffer per
    node group (ZNN_KEEP_IMAGES=1), bit for bit."""
    cfg, params, x, lab = _case("c4", 16, (2, 2, 2))
    xd, ld = torch.as_tensor(x, device="cuda"), torch.as_tensor(lab, device="cuda")
    out = []
    for keep in ("0", "1"):
        monkeypatch.setenv("ZNN_KEEP_IMAGES", keep)
        net = _net(ctx, cfg, params)
        ls = [net.train_step(xd, ld) for _ in range(2)]
        out.append((ls, net.get_params(), net.get_gradients()))
        net.close()
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1]) and np.array_equal(out[0][2], out[1][2])


def test_loader_from_znnv_directory_matches_step_host(ctx, tmp_path):
    """Data provider over ZNNV files (inputs/ + labels/, sorted pairs, the
    same volume into every input / output node): steps through the loader ==
    step_host on the same batches."""
    from paper_1510_06706_b200 import Loader, configs as C, read_volume, write_volume
    cfg = C.scaled("c4", 16, (2, 2, 2), batch=2)
    rng = np.random.default_rng(8)
    params = C.init_params(cfg, 8)
    S = 3  # samples; batch 2 -> steps wrap around (sample index mod 3)
    xs = rng.uniform(0, 1, size=(S,) + tuple(cfg.in_dims)).astype(np.float32)
    ys = (rng.uniform(size=(S,) + tuple(cfg.out_dims)) < 0.5).astype(np.float32)
    os.makedirs(tmp_path / "inputs")
    os.makedirs(tmp_path / "labels")
    for i in range(S):
        write_volume(str(tmp_path / "inputs" / f"s{i:03d}.znnv"), xs[i])
        write_volume(str(tmp_path / "labels" / f"s{i:03d}.znnv"), ys[i])
        assert np.array_equal(read_volume(str(tmp_path / "inputs" / f"s{i:03d}.znnv")), xs[i])
    nout = cfg.layers[-1].width
    a = _net(ctx, cfg, params)
    ld = Loader(a, directory=str(tmp_path))
    assert len(ld) == S
    b = _net(ctx, cfg, params)
    for t in range(4):
        idx = [(t * 2 + j) % S for j in range(2)]
        xin = xs[idx][:, None]
        lab = np.repeat(ys[idx][:, None], nout, axis=1)
        lb = b.step_host(xin, lab)
        la = a.step_loader(ld)
        assert la == lb, (t, la, lb)
    assert np.array_equal(a.get_params(), b.get_params())
    ld.close()


def test_loader_from_pinned_host_arrays(ctx):
    from paper_1510_06706_b200 import Loader
    cfg, params, x, lab = _case("c4", 16, (2, 2, 2))
    xs = torch.from_numpy(x).pin_memory()
    ys = torch.from_numpy(lab).pin_memory()
    a, b = _net(ctx, cfg, params), _net(ctx, cfg, params)
    ld = Loader(a, inputs=xs, labels=ys)
    for _ in range(3):
        assert a.step_loader(ld) == b.step_host(x, lab)
    assert np.array_equal(a.get_params(), b.get_params())


def test_dp_step_single_rank_matches_train_step(ctx):
    """znn_net_train_step_dp over a one-rank NCCL communicator (per-layer
    allreduce buckets on the communication stream, then the update) ==
    the single-process fused step."""
    from paper_1510_06706_b200 import Comm, comm_unique_id
    cfg, params, x, lab = _case()
    xd, ld = torch.as_tensor(x, device="cuda"), torch.as_tensor(lab, device="cuda")
    comm = Comm(ctx, comm_unique_id(), 1, 0)
    a, b = _net(ctx, cfg, params), _net(ctx, cfg, params)
    for _ in range(2):
        la = a.train_step_dp(comm, xd, ld)
        lb = b.train_step(xd, ld)
        assert abs(la - lb) <= 1e-6 * abs(lb)
    assert np.array_equal(a.get_params(), b.get_params())
    t = torch.arange(1000, device="cuda", dtype=torch.float32)
    comm.allreduce(t)
    torch.cuda.synchronize()
    assert torch.equal(t, torch.arange(1000, device="cuda", dtype=torch.float32))
    comm.close()


def test_autotune_layer_entry_point(ctx):
    """trainer.hpp:181-250 per signature: c4 conv2 (80 -> 80, 7^3, s2) at B=8
    goes FFT; a thin 3^3 layer reports all three timings and picks the fastest."""
    from paper_1510_06706_b200 import autotune_layer
    eng, t = autotune_layer(ctx, 8, 80, 80, (62, 62, 62), (7, 7, 7), (2, 2, 2), trials=1)
    assert eng == "fft" and t["fft"] < t["direct"], t
    # thin 16 -> 16 layer: all three engines are candidates (tcgen05 needs >= 16 maps)
    eng, t = autotune_layer(ctx, 1, 16, 16, (18, 18, 18), (3, 3, 3), trials=1)
    assert set(t) == {"direct", "fft", "simt"} and eng == min(t, key=t.get), (eng, t)


@pytest.mark.slow
def test_c5_full_step_leaves_headroom(stream_ctx):
    """The bench configuration (c5, B=16, autotuned) plans its spectra from
    cudaMemGetInfo and leaves >= 20 GB of device memory free after a step."""
    from paper_1510_06706_b200 import Net, configs as C, mem_stats
    ctx, st = stream_ctx
    cfg = C.CONFIGS["c5"]
    net = Net(ctx, cfg.netspec(), cfg.out_dims, batch=cfg.batch, lr=cfg.lr, momentum=cfg.momentum,
              loss=cfg.loss)
    for li in (1, 2, 3, 4):
        net.set_layer_engine(li, "fft")
    net.set_params(C.init_params(cfg, 1))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(0)
    x = torch.rand((16, 1) + tuple(cfg.in_dims), device="cuda", generator=gen)
    lab = (torch.rand((16, 3) + tuple(cfg.out_dims), device="cuda", generator=gen) < 0.5).float()
    torch.cuda.synchronize()
    l0 = net.train_step(x, lab)
    l1 = net.train_step(x, lab)
    assert np.isfinite(l0) and np.isfinite(l1)
    free_gb = mem_stats(ctx)["free"] / 2**30
    torch_cached = torch.cuda.memory_reserved() / 2**30
    assert free_gb + torch_cached >= 20.0, (free_gb, torch_cached)
    net.close()
