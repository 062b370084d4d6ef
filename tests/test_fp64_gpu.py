"""NF_MATH_FP64 (the paper's real64 build) against the fp64 oracle (-m gpu).

The double path computes in fp64 end to end and rounds once to fp32 at the ABI, so its bar
(FP64_BAR, reading R19) is a few fp32 ulps: tighter than the fp32 path can reach, which the
last test checks so the bar cannot be met by accident.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from parity import FP64_BAR, rel_err

pytestmark = pytest.mark.gpu

import paper_1902_06714_b200 as nf  # noqa: E402

SHAPES = [
    ([3, 5, 2], "sigmoid", 8),
    ([37, 45, 13], "tanh", 77),
    ([784, 30, 10], "sigmoid", 1000),
    ([64, 33, 129, 7], "relu,sigmoid", 130),
    ([20, 200, 150, 5], "gaussian", 67),
    ([300, 260, 1], "tanh,relu", 300),
    ([1, 1], "sigmoid", 1),
    ([516, 132, 7], "sigmoid", 1031),
]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def make_net(dims, act, params):
    """fp32 parameters (exactly representable), then the double mode: the oracle sees the
    same values widened."""
    net = nf.Net(dims, act)
    net.set_params(dev(params.astype(np.float32)))
    net.set_math(nf.NF_MATH_FP64)
    return net


def eta32(v):
    """The ABI takes eta as fp32: hand the oracle the same value."""
    return float(np.float32(v))


def f32(p):
    return p.astype(np.float32).astype(np.float64)


def gpu_params(net):
    out = torch.empty(net.n_params, dtype=torch.float32, device="cuda")
    net.get_params(out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("dims,act,n", SHAPES)
def test_fp64_output(dims, act, n):
    p = f32(synth.random_params(len(dims) * 7 + n, dims, 0.5))
    x, _ = synth.random_batch(n, n, dims[0], dims[-1], "normal")
    out = make_net(dims, act, p).output(dev(x)).cpu().numpy()
    assert rel_err(out, oracle.Oracle(dims, act).output(p, x)) <= FP64_BAR


@pytest.mark.parametrize("dims,act,n", SHAPES)
def test_fp64_grad(dims, act, n):
    p = f32(synth.random_params(len(dims) * 11 + n, dims, 0.5))
    x, y = synth.random_batch(n + 1, n, dims[0], dims[-1], "uniform")
    g = make_net(dims, act, p).grad(dev(x), dev(y)).cpu().numpy()
    o = oracle.Oracle(dims, act)
    for (Wg, bg), (Wr, br) in zip(o.layers(g), o.layers(o.grad(p, x, y))):
        assert rel_err(Wg, Wr) <= FP64_BAR
        assert rel_err(bg, br) <= FP64_BAR


@pytest.mark.parametrize("dims,act,n", SHAPES)
def test_fp64_train_batch(dims, act, n):
    p = f32(synth.random_params(len(dims) * 13 + n, dims, 0.5))
    x, y = synth.random_batch(n + 2, n, dims[0], dims[-1], "uniform")
    net = make_net(dims, act, p)
    net.train_batch(dev(x), dev(y), 0.7)
    ref, _ = oracle.Oracle(dims, act).train_batch(p, x, y, eta32(0.7))
    assert rel_err(gpu_params(net), ref) <= FP64_BAR


def test_fp64_split_k_gradient():
    """Batch 5000 rows: the gradient GEMM takes the split-K path (partials + reduce)."""
    dims = [200, 64, 10]
    p = f32(synth.random_params(3, dims, 0.3))
    x, y = synth.random_batch(4, 5000, dims[0], dims[-1], "uniform")
    g = make_net(dims, "sigmoid", p).grad(dev(x), dev(y)).cpu().numpy()
    assert rel_err(g, oracle.Oracle(dims, "sigmoid").grad(p, x, y)) <= FP64_BAR


def test_fp64_c1_full_trajectory():
    cfg = synth.CONFIGS[1]
    p = f32(synth.init_params(1))
    X, Y = synth.dataset(1)
    starts = synth.batch_starts(1)
    net = make_net(cfg["dims"], cfg["act"], p)
    loss = torch.zeros(len(starts), device="cuda")
    net.train_steps(dev(X), dev(Y), cfg["batch"], starts, cfg["eta"], step_loss=loss)
    ref, ref_loss = oracle.Oracle(cfg["dims"], cfg["act"]).train_steps(p, X, Y, cfg["batch"], starts, cfg["eta"])
    assert rel_err(gpu_params(net), ref) <= FP64_BAR
    assert rel_err(loss.cpu().numpy(), ref_loss) <= FP64_BAR


def test_fp64_c2_free_running_200_steps_and_fp32_cannot_match():
    """Config 2 at full size, 200 free-running steps (4 epochs) in double: within a few fp32
    ulps of the oracle trajectory -- the fp32 path on the same run is far outside that bar."""
    cfg = synth.CONFIGS[2]
    p = f32(synth.init_params(2))
    X, Y = synth.dataset(2)
    starts = synth.batch_starts(2)[:200]
    ref, ref_loss = oracle.Oracle(cfg["dims"], cfg["act"]).train_steps(p, X, Y, cfg["batch"], starts, cfg["eta"])
    net = make_net(cfg["dims"], cfg["act"], p)
    loss = torch.zeros(len(starts), device="cuda")
    net.train_steps(dev(X), dev(Y), cfg["batch"], starts, cfg["eta"], step_loss=loss)
    err64 = rel_err(gpu_params(net), ref)
    n32 = nf.Net(cfg["dims"], cfg["act"])
    n32.set_params(dev(p.astype(np.float32)))
    n32.train_steps(dev(X), dev(Y), cfg["batch"], starts, cfg["eta"])
    err32 = rel_err(gpu_params(n32), ref)
    print(f"c2 200 steps: fp64 mode err {err64:.3e}, fp32 mode err {err32:.3e}")
    assert err64 <= FP64_BAR
    assert rel_err(loss.cpu().numpy(), ref_loss) <= FP64_BAR
    assert err32 > 10 * err64


def test_fp64_loss_accuracy():
    dims = [784, 30, 10]
    p = f32(synth.init_params(2))
    X, Y = synth.dataset(2, N=10000)
    net = make_net(dims, "sigmoid", p)
    o = oracle.Oracle(dims, "sigmoid")
    assert abs(net.loss(dev(X), dev(Y)) - o.loss(p, X, Y)) <= FP64_BAR * o.loss(p, X, Y)
    assert abs(net.accuracy(dev(X), dev(Y)) - o.accuracy(p, X, Y)) <= 1e-7


def test_fp64_mode_switch_round_trip():
    """Entering the mode widens exactly (get_params returns the fp32 values bit for bit); a
    step in double then leaving the mode rounds the double parameters into the fp32 arena;
    host and device buffers agree."""
    dims = [37, 45, 13]
    p = synth.random_params(5, dims, 0.5).astype(np.float32)
    x, y = synth.random_batch(5, 50, 37, 13)
    net = make_net(dims, "tanh", p)
    assert np.array_equal(gpu_params(net), p)
    assert np.array_equal(net.get_params(), p)                 # host destination
    net.train_batch(x, y, 0.5)                                 # host inputs
    in_mode = gpu_params(net)
    ref, _ = oracle.Oracle(dims, "tanh").train_batch(p.astype(np.float64), x, y, eta32(0.5))
    assert rel_err(in_mode, ref) <= FP64_BAR
    net.set_math(nf.NF_MATH_FP32)
    assert np.array_equal(gpu_params(net), in_mode)
    net.set_math(nf.NF_MATH_FP64)
    net.set_params(p)                                          # host source, widened
    assert np.array_equal(gpu_params(net), p)
    with pytest.raises(nf.NFError):
        net.set_math(3)


def test_fp64_graph_replay_and_eta_zero():
    """train_steps replays its CUDA graph on a repeated call in double too; eta = 0 leaves the
    parameters bit for bit."""
    dims = [64, 33, 129, 7]
    p = f32(synth.random_params(9, dims, 0.4))
    X, Y = synth.random_batch(10, 300, dims[0], dims[-1], "uniform")
    starts = [0, 100, 200, 50]
    a = make_net(dims, "tanh,sigmoid", p)
    a.train_steps(dev(X), dev(Y), 100, starts, 0.0)
    assert np.array_equal(gpu_params(a), p.astype(np.float32))
    Xd, Yd = dev(X), dev(Y)
    a.train_steps(Xd, Yd, 100, starts, 0.3)
    a.train_steps(Xd, Yd, 100, starts, 0.3)                   # replay
    ref, _ = oracle.Oracle(dims, "tanh,sigmoid").train_steps(p, X, Y, 100, starts + starts, eta32(0.3))
    assert rel_err(gpu_params(a), ref) <= FP64_BAR
