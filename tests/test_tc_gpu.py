"""GPU parity of the tcgen05 tensor-core contractions (gemm_tc.cuh) through the C-ABI (-m gpu).

Shapes are chosen so that every contraction with all extents >= 64 takes the tensor-core
path: K1 (both operands K-major), K3 (B operand N-major), K4 (both operands MN-major),
with ragged tile tails in M, N and K and split-K over the batch.  NF_MATH_FP32 runs them
as 3xTF32 (bar 1e-4 at tau=0.1), NF_MATH_TF32 as 1xTF32 on round-to-nearest TF32 operands
(bar 5e-3 normwise, tau=1: reading R14b of DESIGN.md), both against the fp64 oracle.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from parity import FP32_BAR, TF32_BAR, argmax_agree, rel_err

pytestmark = pytest.mark.gpu

import paper_1902_06714_b200 as nf  # noqa: E402

TC_SHAPES = [
    ([200, 136, 72, 5], "tanh", 300),          # ragged M/N/K tails in every GEMM
    ([256, 128, 64], "sigmoid", 4096),         # K4: few tiles, K = 4096 -> split-K
    ([516, 260, 132, 3], "gaussian,sigmoid", 333),
    ([784, 1024, 1024, 10], "tanh", 256),      # config-3 widths
]


@pytest.fixture(autouse=True, params=["tcgen05", "hmma"])
def engine(request, monkeypatch):
    """Every test runs on both tensor-core engines: tcgen05 (the default) and the opt-in warp-level
    MMA GEMM (gemm_hmma.cuh, NF_HMMA=1: the contractions of <= 2 GFLOP)."""
    if request.param == "hmma":
        monkeypatch.setenv("NF_HMMA", "1")
    else:
        monkeypatch.delenv("NF_HMMA", raising=False)
    return request.param


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check(got, ref, math):
    if math == nf.NF_MATH_FP32:
        assert rel_err(got, ref) <= FP32_BAR
    else:
        assert rel_err(got, ref, tau=1.0) <= TF32_BAR


def make_net(dims, act, params, math):
    net = nf.Net(dims, act)
    net.set_math(math)
    net.set_params(dev(params.astype(np.float32)))
    return net


def gpu_params(net):
    out = torch.empty(net.n_params, dtype=torch.float32, device="cuda")
    net.get_params(out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("math,bar", [(nf.NF_MATH_FP32, FP32_BAR), (nf.NF_MATH_TF32, TF32_BAR)])
@pytest.mark.parametrize("dims,act,n", TC_SHAPES)
def test_tc_output(dims, act, n, math, bar):
    p = synth.random_params(len(dims) * 3 + n, dims, 1.0 / np.sqrt(max(dims)))
    x, _ = synth.random_batch(n, n, dims[0], dims[-1], "normal")
    net = make_net(dims, act, p, math)
    out = net.output(dev(x)).cpu().numpy()
    ref = oracle.Oracle(dims, act).output(p, x)
    check(out, ref, math)
    if math == nf.NF_MATH_FP32:
        assert argmax_agree(out, ref)[0] == 0


@pytest.mark.parametrize("math,bar", [(nf.NF_MATH_FP32, FP32_BAR), (nf.NF_MATH_TF32, TF32_BAR)])
@pytest.mark.parametrize("dims,act,n", TC_SHAPES)
def test_tc_grad(dims, act, n, math, bar):
    p = synth.random_params(len(dims) * 5 + n, dims, 1.0 / np.sqrt(max(dims)))
    x, y = synth.random_batch(n + 3, n, dims[0], dims[-1], "uniform")
    net = make_net(dims, act, p, math)
    g = net.grad(dev(x), dev(y)).cpu().numpy()
    o = oracle.Oracle(dims, act)
    ref = o.grad(p, x, y)
    for (Wg, bg), (Wr, br) in zip(o.layers(g), o.layers(ref)):
        check(Wg, Wr, math)
        check(bg, br, math)


@pytest.mark.parametrize("math,bar", [(nf.NF_MATH_FP32, FP32_BAR), (nf.NF_MATH_TF32, TF32_BAR)])
@pytest.mark.parametrize("dims,act,n", TC_SHAPES[:3])
def test_tc_train_batch(dims, act, n, math, bar):
    p = synth.random_params(len(dims) * 9 + n, dims, 1.0 / np.sqrt(max(dims)))
    x, y = synth.random_batch(n + 4, n, dims[0], dims[-1], "uniform")
    net = make_net(dims, act, p, math)
    net.train_batch(dev(x), dev(y), 0.5)
    o = oracle.Oracle(dims, act)
    ref, _ = o.train_batch(p, x, y, 0.5)
    got = gpu_params(net)
    for (Wg, bg), (Wr, br) in zip(o.layers(got), o.layers(ref)):
        check(Wg, Wr, math)
        check(bg, br, math)
    # the update itself (W' - W) carries the contraction error undiluted by W
    for (Wg, _), (Wr, _), (W0, _) in zip(o.layers(got), o.layers(ref), o.layers(p.astype(np.float64))):
        assert rel_err(Wg - W0, Wr - W0) <= (1e-3 if math == nf.NF_MATH_FP32 else 2e-2)


def test_tc_c5_full_width_grad():
    """Config-5 widths on 64 rows: every layer of K1/K3/K4 at 4096/1024 widths on the
    tensor cores (3xTF32, fp32 mode); rows with relu pre-activations inside the rounding
    band are excluded (R8)."""
    cfg = synth.CONFIGS[5]
    dims = cfg["dims"]
    p = synth.init_params(5)
    X, Y = synth.dataset(5, N=160)
    o = oracle.Oracle(dims, cfg["act"])
    keep = o.kink_free_rows(p, X, Y)
    X, Y = np.ascontiguousarray(X[keep][:64]), np.ascontiguousarray(Y[keep][:64])
    assert len(X) == 64
    net = make_net(dims, cfg["act"], p, nf.NF_MATH_FP32)
    g = net.grad(dev(X), dev(Y)).cpu().numpy()
    ref = o.grad(p, X, Y)
    for (Wg, bg), (Wr, br) in zip(o.layers(g), o.layers(ref)):
        assert rel_err(Wg, Wr) <= FP32_BAR
        assert rel_err(bg, br) <= FP32_BAR


# ------------------------------------------------------------------ full-size launches
@pytest.mark.parametrize("cid,math", [(5, nf.NF_MATH_TF32), (5, nf.NF_MATH_FP32), (3, nf.NF_MATH_TF32),
                                      (3, nf.NF_MATH_FP32), (4, nf.NF_MATH_TF32), (4, nf.NF_MATH_FP32)])
def test_full_batch_forward_sampled_rows(cid, math):
    """nf_output over a full training batch (c5: 16384 rows, the persistent 1xTF32 GEMM in TF32
    mode; c3: 4096 rows) in the launch configuration bench.py times; 16 sampled rows against the
    fp64 oracle (rows the oracle can afford one by one)."""
    cfg = synth.CONFIGS[cid]
    dims = cfg["dims"]
    p = synth.init_params(cid)
    X, _ = synth.dataset(cid, N=cfg["batch"])
    net = make_net(dims, cfg["act"], p, math)
    out = net.output(dev(X)).cpu().numpy()
    rows = np.linspace(0, cfg["batch"] - 1, 16).astype(int)
    ref = oracle.Oracle(dims, cfg["act"]).output(p, np.ascontiguousarray(X[rows]))
    check(out[rows], ref, math)


@pytest.mark.parametrize("cid,math", [(5, nf.NF_MATH_TF32), (3, nf.NF_MATH_TF32), (3, nf.NF_MATH_FP32)])
def test_full_batch_grad_split_invariance(cid, math):
    """The co_sum property at full batch size: the tendencies of the whole batch equal
    the sum over its two halves, all on the GPU in the bench's launch configuration."""
    cfg = synth.CONFIGS[cid]
    dims, B = cfg["dims"], cfg["batch"]
    p = synth.init_params(cid)
    X, Y = synth.dataset(cid, N=B)
    net = make_net(dims, cfg["act"], p, math)
    g = net.grad(dev(X), dev(Y)).cpu().numpy().astype(np.float64)
    g1 = net.grad(dev(X[:B // 2]), dev(Y[:B // 2])).cpu().numpy().astype(np.float64)
    g2 = net.grad(dev(X[B // 2:]), dev(Y[B // 2:])).cpu().numpy().astype(np.float64)
    o = oracle.Oracle(dims, cfg["act"])
    for (Wa, ba), (Wb, bb) in zip(o.layers(g), o.layers(g1 + g2)):
        check(Wa, Wb, math)
        check(ba, bb, math)


def test_transposed_gradient_operands(monkeypatch, engine):
    """NF_TPOSE=1 (opt-in since the warp-uniform MMA issue): the forward / delta epilogues also store
    A_l^T / delta_l^T so that the weight-gradient contraction reads K-major operands (store_t, the
    K/K persistent EpiGrad).  One TF32 SGD step at config-5 widths (a wave or more of 128 x 256
    tiles per GEMM) against the batched fp64 oracle, tanh hidden layers (reading R20)."""
    if engine != "tcgen05":
        pytest.skip("tcgen05 path only")
    from oracle.batched import BatchedOracle
    monkeypatch.setenv("NF_TPOSE", "1")
    dims, act, B = [4096, 4096, 4096, 1024], "tanh,sigmoid", 2048
    p = synth.init_params(5, dims)
    X, Y = synth.dataset(5, N=B)
    X = np.ascontiguousarray(X[:, :dims[0]])
    Y = np.ascontiguousarray(Y[:, :dims[-1]])
    o = BatchedOracle(dims, act)
    eta = 5.0
    ref, _, _ = o.train_batch(p, X, Y, eta)
    net = make_net(dims, act, p, nf.NF_MATH_TF32)
    nf.nf_debug_log_enable(True)
    net.train_steps(dev(X), dev(Y), B, [0], eta)
    torch.cuda.synchronize()
    log = nf.nf_debug_log_read()
    nf.nf_debug_log_enable(False)
    # the K-major / K-major weight-gradient instantiation ran (MN / MN without the transposed copies)
    assert any("gemm_tc_persistent<256, false, false, nf::EpiGrad" in l.replace("(bool)0", "false").replace("<256, 0, 0,", "<256, false, false,")
               for l in log), log
    got = gpu_params(net)
    for (Wg, bg), (Wr, br), (W0, b0) in zip(o.layers(got), o.layers(ref), o.layers(p.astype(np.float64))):
        assert rel_err(Wg - W0, Wr - W0, tau=1.0) <= TF32_BAR
        assert rel_err(bg - b0, br - b0, tau=1.0) <= TF32_BAR
