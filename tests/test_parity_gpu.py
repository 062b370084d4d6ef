"""GPU parity of the CUDA path (through the C-ABI) against the fp64 CPU oracle (-m gpu).

Every input comes from synth/ (seeded); every expected value from oracle/.  Bars and the
metric are in tests/parity.py (R14/R15).  Shapes span several tiles with ragged tails;
the full-size configs are checked in the launch configuration bench.py times, on
samples the oracle can compute (teacher-forced steps, sampled rows).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from parity import FP32_BAR, argmax_agree, rel_err

pytestmark = pytest.mark.gpu

import paper_1902_06714_b200 as nf  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def make_net(dims, act, params):
    net = nf.Net(dims, act)
    net.set_params(dev(params.astype(np.float32)))
    return net


def gpu_params(net):
    out = torch.empty(net.n_params, dtype=torch.float32, device="cuda")
    net.get_params(out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


SHAPES = [
    ([3, 5, 2], "sigmoid", 8),
    ([37, 45, 13], "tanh", 77),
    ([784, 30, 10], "sigmoid", 1000),
    ([64, 33, 129, 7], "relu,sigmoid", 130),
    ([20, 200, 150, 5], "gaussian", 67),
    ([300, 260, 1], "tanh,relu", 300),
    ([1, 1], "sigmoid", 1),
    ([5, 1, 3], "step,sigmoid", 9),
    # narrow output layers over >= 512 rows: the dedicated skinny kernels (fwd_smalln,
    # bwd_smallk, grad_smallm in kernels.cu)
    ([300, 200, 10], "tanh,sigmoid", 600),
    ([516, 132, 7], "sigmoid", 1031),
    # narrow output layer (n_L <= 16) after a hidden layer of 128..2048 (multiple of 4) over
    # >= 256 rows: the fused output-layer training kernel (out_layer_train: 4-, 8- and 16-slot
    # variants; n_L = 1, 10, 12, 16)
    ([40, 1100, 12], "tanh,sigmoid", 300),
    ([64, 256, 16], "sigmoid", 513),
    ([30, 640, 10], "gaussian,sigmoid", 257),
    # register-resident form (out_layer_train_rg: H % 128 == 0, H <= 1024): 8 row groups of one
    # warp (H = 128), 2 groups with idle threads (H = 384), ragged last iteration
    ([50, 128, 1], "tanh,sigmoid", 389),
    ([70, 384, 16], "relu,sigmoid", 1001),
    # one activation per layer: generic kernels, fused output layer
    ([20, 50, 40, 30, 6], "tanh,gaussian,sigmoid,tanh", 150),
    ([24, 130, 96, 10], "sigmoid,tanh,sigmoid", 300),
    # two-layer nets with narrow layers and n0 % 4 == 0: the fused inference kernel
    # (infer_small.cu) with a ragged last 64-row tile and a ragged last pixel chunk
    ([100, 17, 3], "tanh,sigmoid", 777),
]


@pytest.mark.parametrize("dims,act,n", SHAPES)
def test_output_parity(dims, act, n):
    p = synth.random_params(len(dims) * 7 + n, dims, 0.5)
    x, _ = synth.random_batch(n, n, dims[0], dims[-1], "normal")
    net = make_net(dims, act, p)
    out = net.output(dev(x)).cpu().numpy()
    ref = oracle.Oracle(dims, act).output(p, x)
    assert rel_err(out, ref) <= FP32_BAR
    mism, _ = argmax_agree(out, ref)
    assert mism == 0


@pytest.mark.parametrize("dims,act,n", SHAPES)
def test_grad_parity(dims, act, n):
    p = synth.random_params(len(dims) * 11 + n, dims, 0.5)
    x, y = synth.random_batch(n + 1, n, dims[0], dims[-1], "uniform")
    net = make_net(dims, act, p)
    g = net.grad(dev(x), dev(y)).cpu().numpy()
    ref = oracle.Oracle(dims, act).grad(p, x, y)
    o = oracle.Oracle(dims, act)
    for (Wg, bg), (Wr, br) in zip(o.layers(g), o.layers(ref)):
        assert rel_err(Wg, Wr) <= FP32_BAR
        assert rel_err(bg, br) <= FP32_BAR


@pytest.mark.parametrize("dims,act,n", SHAPES)
def test_train_batch_parity(dims, act, n):
    p = synth.random_params(len(dims) * 13 + n, dims, 0.5)
    x, y = synth.random_batch(n + 2, n, dims[0], dims[-1], "uniform")
    net = make_net(dims, act, p)
    net.train_batch(dev(x), dev(y), 0.7)
    got = gpu_params(net)
    ref, _ = oracle.Oracle(dims, act).train_batch(p, x, y, 0.7)
    o = oracle.Oracle(dims, act)
    # compare the update itself (params move little; the update is what the step computes)
    for (Wg, bg), (Wr, br), (W0, b0) in zip(o.layers(got), o.layers(ref), o.layers(p.astype(np.float64))):
        assert rel_err(Wg, Wr) <= FP32_BAR
        assert rel_err(Wg - W0, Wr - W0) <= 1e-3   # fp32 cancellation of W - W0 bounds this
        assert rel_err(bg, br) <= FP32_BAR


def test_eta_zero_is_bitwise_noop():
    dims = [784, 30, 10]
    p = synth.init_params(2)
    X, Y = synth.dataset(2, N=2000)
    net = make_net(dims, "sigmoid", p)
    net.train_batch(dev(X[:1000]), dev(Y[:1000]), 0.0)
    assert np.array_equal(gpu_params(net), p)
    net.train_steps(dev(X), dev(Y), 1000, [0, 500, 1000], 0.0)   # fused path
    assert np.array_equal(gpu_params(net), p)


def test_split_batch_co_sum_on_gpu():
    """tendencies of a batch == sum over any split (the co_sum property)."""
    dims = [784, 30, 10]
    p = synth.init_params(2)
    X, Y = synth.dataset(2, N=1000)
    net = make_net(dims, "sigmoid", p)
    g = net.grad(dev(X), dev(Y)).cpu().numpy().astype(np.float64)
    g1 = net.grad(dev(X[:377]), dev(Y[:377])).cpu().numpy().astype(np.float64)
    g2 = net.grad(dev(X[377:]), dev(Y[377:])).cpu().numpy().astype(np.float64)
    assert rel_err(g1 + g2, g) <= FP32_BAR


def test_loss_accuracy_parity():
    dims = [784, 30, 10]
    p = synth.init_params(2)
    X, Y = synth.dataset(2, N=10000)
    net = make_net(dims, "sigmoid", p)
    o = oracle.Oracle(dims, "sigmoid")
    assert abs(net.loss(dev(X), dev(Y)) - o.loss(p, X, Y)) <= FP32_BAR * o.loss(p, X, Y)
    out = net.output(dev(X)).cpu().numpy()
    ref = o.output(p, X)
    mism, ties = argmax_agree(out, ref)
    assert mism == 0
    acc_ref = o.accuracy(p, X, Y)
    assert abs(net.accuracy(dev(X), dev(Y)) - acc_ref) <= ties / len(X) + 1e-7
    assert 0.05 < acc_ref < 0.15          # untrained net = chance


def test_degenerate_inputs():
    net = make_net([4, 3, 2], "sigmoid", synth.random_params(1, [4, 3, 2]))
    assert net.accuracy(dev(np.zeros((0, 4), np.float32)), dev(np.zeros((0, 2), np.float32))) == 0.0
    out = torch.empty((0, 2), device="cuda")
    nf.nf_output(net.h, dev(np.zeros((1, 4), np.float32)), 0, out)
    with pytest.raises(nf.NFError):
        nf.nf_train_batch(net.h, dev(np.zeros((1, 4), np.float32)), dev(np.zeros((1, 2), np.float32)), 0, 1.0)
    with pytest.raises(nf.NFError):
        nf.nf_train_batch(net.h, dev(np.zeros((1, 4), np.float32)), dev(np.zeros((1, 2), np.float32)), 1,
                          float("nan"))


def test_host_pointers_match_device_pointers():
    dims = [37, 45, 13]
    p = synth.random_params(5, dims, 0.5)
    x, y = synth.random_batch(5, 50, 37, 13)
    a = make_net(dims, "tanh", p)
    b = make_net(dims, "tanh", p)
    a.train_batch(x, y, 0.5)                      # numpy host buffers
    b.train_batch(dev(x), dev(y), 0.5)
    assert np.array_equal(gpu_params(a), gpu_params(b))
    assert np.array_equal(a.output(x), b.output(dev(x)).cpu().numpy())
    assert np.array_equal(a.grad(x, y), b.grad(dev(x), dev(y)).cpu().numpy())


# ------------------------------------------------------------------ full configs
def test_c1_full_trajectory():
    """Config 1 in full: [3,5,2] sigmoid, 64 samples, B=8, eta=1, 100 steps (fused kernel)."""
    cfg = synth.CONFIGS[1]
    p = synth.init_params(1)
    X, Y = synth.dataset(1)
    starts = synth.batch_starts(1)
    net = make_net(cfg["dims"], cfg["act"], p)
    loss = torch.zeros(len(starts), device="cuda")
    net.train_steps(dev(X), dev(Y), cfg["batch"], starts, cfg["eta"], step_loss=loss)
    ref, ref_loss = oracle.Oracle(cfg["dims"], cfg["act"]).train_steps(p, X, Y, cfg["batch"], starts, cfg["eta"])
    assert rel_err(gpu_params(net), ref) <= FP32_BAR
    assert rel_err(loss.cpu().numpy(), ref_loss) <= FP32_BAR


def test_c1_generic_path_equals_fused_semantics():
    """The per-step kernels (nf_train_batch loop) and the fused kernel agree."""
    cfg = synth.CONFIGS[1]
    p = synth.init_params(1)
    X, Y = synth.dataset(1)
    starts = synth.batch_starts(1, steps=20)
    a = make_net(cfg["dims"], cfg["act"], p)
    b = make_net(cfg["dims"], cfg["act"], p)
    a.train_steps(dev(X), dev(Y), 8, starts, 1.0)
    for s in starts:
        b.train_batch(dev(X[s:s + 8]), dev(Y[s:s + 8]), 1.0)
    assert rel_err(gpu_params(a), gpu_params(b)) <= FP32_BAR


@pytest.fixture(scope="module")
def c2_trajectory():
    """Oracle (fp64) run of config 2 in full: 500 steps, with fp32-rounded checkpoints."""
    cfg = synth.CONFIGS[2]
    p0 = synth.init_params(2)
    X, Y = synth.dataset(2)
    starts = synth.batch_starts(2)
    o = oracle.Oracle(cfg["dims"], cfg["act"])
    ckpt = {}
    p = p0.astype(np.float64)
    losses = []
    for a, b in [(0, 100), (100, 250), (250, 490), (490, 500)]:
        ckpt[a] = p.astype(np.float32)
        p, l = o.train_steps(p, X, Y, cfg["batch"], starts[a:b], cfg["eta"])
        losses.append(l)
    ckpt[500] = p
    return dict(cfg=cfg, X=X, Y=Y, starts=starts, ckpt=ckpt, p0=p0, loss=np.concatenate(losses))


@pytest.mark.parametrize("at", [0, 100, 250, 490])
def test_c2_teacher_forced_steps(c2_trajectory, at):
    """Config 2 at full size, fused kernel in the bench's launch configuration: from the
    oracle's fp32-rounded parameters at step `at`, 10 GPU steps vs 10 oracle steps."""
    t = c2_trajectory
    cfg, X, Y = t["cfg"], t["X"], t["Y"]
    starts = t["starts"][at:at + 10]
    p = t["ckpt"][at]
    net = make_net(cfg["dims"], cfg["act"], p)
    Xd, Yd = dev(X), dev(Y)
    loss = torch.zeros(len(starts), device="cuda")
    net.train_steps(Xd, Yd, cfg["batch"], starts, cfg["eta"], step_loss=loss)
    o = oracle.Oracle(cfg["dims"], cfg["act"])
    ref, ref_loss = o.train_steps(p, X, Y, cfg["batch"], starts, cfg["eta"])
    got = gpu_params(net)
    for (Wg, bg), (Wr, br) in zip(o.layers(got), o.layers(ref)):
        assert rel_err(Wg, Wr) <= FP32_BAR
        assert rel_err(bg, br) <= FP32_BAR
    assert rel_err(loss.cpu().numpy(), ref_loss) <= FP32_BAR


def test_c2_single_step_gradient_full_size(c2_trajectory):
    """One full-size c2 step: the applied update (W_after - W_before) against the oracle's."""
    t = c2_trajectory
    cfg, X, Y = t["cfg"], t["X"], t["Y"]
    s = int(t["starts"][0])
    p = t["p0"]
    net = make_net(cfg["dims"], cfg["act"], p)
    net.train_steps(dev(X), dev(Y), cfg["batch"], [s], cfg["eta"])
    o = oracle.Oracle(cfg["dims"], cfg["act"])
    g = o.grad(p, X[s:s + 1000], Y[s:s + 1000]) * (cfg["eta"] / 1000)
    upd = p.astype(np.float64) - gpu_params(net).astype(np.float64)
    for (Ug, ub), (Ur, br) in zip(o.layers(upd), o.layers(g)):
        assert rel_err(Ug, Ur) <= 5e-3   # W - W' in fp32 loses ~|W|/|dW| * 2^-24 relative
        assert rel_err(ub, br) <= 5e-3


def test_c2_free_running_500_steps(c2_trajectory):
    """Whole config 2 (10 epochs) free-running on the GPU vs the fp64 oracle trajectory.
    Reported bar 1e-3 on the final parameters, plus the per-step losses."""
    t = c2_trajectory
    cfg = t["cfg"]
    net = make_net(cfg["dims"], cfg["act"], t["p0"])
    loss = torch.zeros(500, device="cuda")
    net.train_steps(dev(t["X"]), dev(t["Y"]), cfg["batch"], t["starts"], cfg["eta"], step_loss=loss)
    err = rel_err(gpu_params(net), t["ckpt"][500])
    print(f"c2 free-running final-param err {err:.3e}")
    assert err <= 1e-3
    assert rel_err(loss.cpu().numpy(), t["loss"]) <= 1e-3


def test_c5_full_width_sampled():
    """Config 5 widths [4096,4096,4096,4096,1024]: forward on sampled rows and one-step
    tendencies on a small batch (the oracle's per-sample cost is batch independent)."""
    cfg = synth.CONFIGS[5]
    dims = cfg["dims"]
    p = synth.init_params(5)
    X, Y = synth.dataset(5, N=64)
    net = make_net(dims, cfg["act"], p)
    o = oracle.Oracle(dims, cfg["act"])
    rows = np.arange(0, 64, 8)
    out = net.output(dev(X)).cpu().numpy()
    assert rel_err(out[rows], o.output(p, X[rows])) <= FP32_BAR
    g = net.grad(dev(X[:6]), dev(Y[:6])).cpu().numpy()
    ref = o.grad(p, X[:6], Y[:6])
    for (Wg, bg), (Wr, br) in zip(o.layers(g), o.layers(ref)):
        assert rel_err(Wg, Wr) <= FP32_BAR
        assert rel_err(bg, br) <= FP32_BAR


@pytest.mark.parametrize("cid,n", [(3, 64), (4, 256)])
def test_c3_c4_full_width_one_step(cid, n):
    """One step at the full widths of configs 3 and 4.  Rows with a relu pre-activation
    inside the fp32 rounding band (|z| <= 1e-4) are excluded: there relu' is a discrete
    decision both sides may take differently (R8); the rest must match to 1e-4 per layer."""
    cfg = synth.CONFIGS[cid]
    dims = cfg["dims"]
    p = synth.init_params(cid)
    X, Y = synth.dataset(cid, N=n)
    o = oracle.Oracle(dims, cfg["act"])
    keep = o.kink_free_rows(p, X, Y)
    assert keep.mean() > 0.5
    X, Y = np.ascontiguousarray(X[keep]), np.ascontiguousarray(Y[keep])
    net = make_net(dims, cfg["act"], p)
    net.train_batch(dev(X), dev(Y), cfg["eta"])
    ref, _ = o.train_batch(p, X, Y, cfg["eta"])
    for (Wg, bg), (Wr, br) in zip(o.layers(gpu_params(net)), o.layers(ref)):
        assert rel_err(Wg, Wr) <= FP32_BAR
        assert rel_err(bg, br) <= FP32_BAR


@pytest.mark.parametrize("engine", ["tc", "ffma2"])
def test_c2_tensor_core_variant_of_fused_kernel(c2_trajectory, monkeypatch, engine):
    """The two contraction engines of the fused kernel on config 2: tcgen05 split-TF32 (the default
    where it applies) and packed FFMA2 (NF_FUSED_TC=0): same parity bar; the launch log shows which
    instantiation ran."""
    monkeypatch.setenv("NF_FUSED_TC", "1" if engine == "tc" else "0")
    nf.nf_debug_log_enable(True)
    t = c2_trajectory
    cfg, X, Y = t["cfg"], t["X"], t["Y"]
    starts = t["starts"][100:110]
    p = t["ckpt"][100]
    net = make_net(cfg["dims"], cfg["act"], p)
    loss = torch.zeros(len(starts), device="cuda")
    net.train_steps(dev(X), dev(Y), cfg["batch"], starts, cfg["eta"], step_loss=loss)
    log = nf.nf_debug_log_read()
    nf.nf_debug_log_enable(False)
    want = "fused_small_kernel<true" if engine == "tc" else "fused_small_kernel<false, false"
    assert any(want in l for l in log), log
    o = oracle.Oracle(cfg["dims"], cfg["act"])
    ref, ref_loss = o.train_steps(p, X, Y, cfg["batch"], starts, cfg["eta"])
    for (Wg, bg), (Wr, br) in zip(o.layers(gpu_params(net)), o.layers(ref)):
        assert rel_err(Wg, Wr) <= FP32_BAR
        assert rel_err(bg, br) <= FP32_BAR
    assert rel_err(loss.cpu().numpy(), ref_loss) <= FP32_BAR


@pytest.mark.parametrize("geom,batch", [({}, 1000), ({"NF_FUSED_C": "7"}, 1000), ({}, 900), ({}, 333)])
def test_c2_warp_mma_variant_of_fused_kernel(c2_trajectory, monkeypatch, geom, batch):
    """The opt-in warp-level MMA (mma.sync 3xTF32) variant of the fused kernel (NF_FUSED_MM=1),
    in the default decomposition (5 row m-tiles, 100-pixel slices), 112-pixel slices (the other row
    permutation of its conflict-free loads), 60-row clusters (4 m-tiles) and ragged 23-row clusters:
    same parity bar."""
    monkeypatch.setenv("NF_FUSED_MM", "1")
    for k, v in geom.items():
        monkeypatch.setenv(k, v)
    nf.nf_debug_log_enable(True)
    t = c2_trajectory
    cfg, X, Y = t["cfg"], t["X"], t["Y"]
    starts = t["starts"][100:110]
    p = t["ckpt"][100]
    net = make_net(cfg["dims"], cfg["act"], p)
    loss = torch.zeros(len(starts), device="cuda")
    net.train_steps(dev(X), dev(Y), batch, starts, cfg["eta"], step_loss=loss)
    torch.cuda.synchronize()
    log = nf.nf_debug_log_read()
    nf.nf_debug_log_enable(False)
    assert any("fused_small_kernel" in l and " mma" in l for l in log), log
    o = oracle.Oracle(cfg["dims"], cfg["act"])
    ref, ref_loss = o.train_steps(p, X, Y, batch, starts, cfg["eta"])
    for (Wg, bg), (Wr, br) in zip(o.layers(gpu_params(net)), o.layers(ref)):
        assert rel_err(Wg, Wr) <= FP32_BAR
        assert rel_err(bg, br) <= FP32_BAR
    assert rel_err(loss.cpu().numpy(), ref_loss) <= FP32_BAR


def test_generic_train_steps_graph_equals_train_batch_loop():
    """nf_train_steps on a generic (non-fused) net runs as a captured CUDA graph, replayed on a
    repeated call; it must equal the nf_train_batch loop, and its replay must equal a fresh run."""
    dims, act, B = [200, 136, 72, 5], "tanh", 128
    p = synth.random_params(31, dims, 0.1)
    X, Y = synth.random_batch(32, 1024, dims[0], dims[-1], "uniform")
    starts = [0, 300, 77, 896, 512]
    a = make_net(dims, act, p)
    b = make_net(dims, act, p)
    a.train_steps(dev(X), dev(Y), B, starts, 0.5)            # capture + launch
    for s in starts:
        b.train_batch(dev(X[s:s + B]), dev(Y[s:s + B]), 0.5)
    # same kernels; only the arrival order of the L2 reductions of the bias tendencies may
    # differ between two runs (reading R12): equal to within fp32 rounding, 10x inside the bar
    assert rel_err(gpu_params(a), gpu_params(b)) <= 1e-5
    n0 = nf.nf_launch_count()
    a.set_params(dev(p))
    a.train_steps(dev(X), dev(Y), B, starts, 0.5)            # replay (same arguments)
    assert nf.nf_launch_count() > n0                          # replays count their kernels
    assert rel_err(gpu_params(a), gpu_params(b)) <= 1e-5
    o = oracle.Oracle(dims, act)
    ref, _ = o.train_steps(p, X, Y, B, starts, 0.5)
    assert rel_err(gpu_params(a), ref) <= FP32_BAR


def test_generic_train_steps_on_a_side_stream():
    dims, act, B = [200, 136, 72, 5], "tanh", 128
    p = synth.random_params(33, dims, 0.1)
    X, Y = synth.random_batch(34, 512, dims[0], dims[-1], "uniform")
    st = torch.cuda.Stream()
    net = nf.Net(dims, act, stream=st)
    net.set_params(dev(p))
    with torch.cuda.stream(st):
        net.train_steps(dev(X), dev(Y), B, [0, 128, 384], 0.5)
    st.synchronize()
    ref, _ = oracle.Oracle(dims, act).train_steps(p, X, Y, B, [0, 128, 384], 0.5)
    out = torch.empty(net.n_params, dtype=torch.float32, device="cuda")
    net.get_params(out)
    st.synchronize()
    assert rel_err(out.cpu().numpy(), ref) <= FP32_BAR


def test_fused_inference_equals_generic_path(monkeypatch):
    """nf_output / nf_loss / nf_accuracy of a small two-layer net: the fused inference kernel
    and the generic K1 chain agree (both against the oracle)."""
    dims = [784, 30, 10]
    p = synth.init_params(2)
    X, Y = synth.dataset(2, N=5000)
    net = make_net(dims, "sigmoid", p)
    fused = net.output(dev(X)).cpu().numpy()
    lf, af = net.loss(dev(X), dev(Y)), net.accuracy(dev(X), dev(Y))
    monkeypatch.setenv("NF_DISABLE_FUSED", "1")
    generic = net.output(dev(X)).cpu().numpy()
    lg, ag = net.loss(dev(X), dev(Y)), net.accuracy(dev(X), dev(Y))
    ref = oracle.Oracle(dims, "sigmoid").output(p, X)
    assert rel_err(fused, ref) <= FP32_BAR and rel_err(generic, ref) <= FP32_BAR
    assert abs(lf - lg) <= 1e-6 * abs(lg) + 1e-9 and af == ag


@pytest.mark.parametrize("dims,act,n", [([784, 30, 10], "sigmoid", 50000), ([784, 30, 10], "sigmoid", 1),
                                        ([784, 30, 10], "sigmoid", 33), ([784, 30, 10], "sigmoid", 4767),
                                        ([100, 17, 3], "tanh,sigmoid", 777), ([64, 32, 32], "relu,tanh", 300),
                                        ([36, 8, 1], "gaussian,sigmoid", 129)])
@pytest.mark.parametrize("form", [0, 1, 2, 3])
def test_tensor_core_inference(dims, act, n, form, monkeypatch):
    """nf_output of two-layer nets with narrow layers on the tcgen05 inference kernels (split TF32,
    infer_tc.cu; form 0 = the default: x from TMEM against W1 hi | lo stacked along N; 1 =
    transposed, three MMAs per k-step; 2 = transposed, W1 hi | lo stacked along M): ragged 32-row
    TMA boxes and 128-row tiles, a ragged last 32-pixel K-block (n0 = 100, 36), every width up to
    32, against the oracle at the fp32 bar; the launch log proves the kernel ran, and the FFMA2
    kernel (NF_INFER_SIMT=1) agrees."""
    monkeypatch.setenv("NF_INFER_TC_FORM", str(form))
    p = synth.random_params(n + 3, dims, 0.5)
    x, _ = synth.random_batch(n + 5, n, dims[0], dims[-1], "uniform")
    net = make_net(dims, act, p)
    nf.nf_debug_log_enable(True)
    out = net.output(dev(x)).cpu().numpy()
    log = nf.nf_debug_log_read()
    nf.nf_debug_log_enable(False)
    assert any(("infer_tc_kernel", "infer_tcT_kernel", "infer_tcS_kernel", "infer_tcX_kernel")[form] in l for l in log), log
    rows = np.arange(n) if n <= 5000 else np.random.default_rng(0).choice(n, 4000, replace=False)
    ref = oracle.Oracle(dims, act).output(p, np.ascontiguousarray(x[rows]))
    assert rel_err(out[rows], ref) <= FP32_BAR
    assert argmax_agree(out[rows], ref)[0] == 0
    monkeypatch.setenv("NF_INFER_SIMT", "1")
    simt = net.output(dev(x)).cpu().numpy()
    assert rel_err(out, simt) <= FP32_BAR


@pytest.mark.parametrize("dims,act", [([784, 30, 10], "sigmoid"), ([3, 5, 2], "sigmoid"),
                                      ([200, 136, 72, 5], "tanh,sigmoid")])
def test_train_single_online_sgd(dims, act):
    """The paper's train_single: batch = 1 steps (online SGD), through nf_train_steps
    (fused kernel for the two-layer nets, the graph of generic kernels otherwise).  The setups are
    well conditioned: the oracle's own fp32 build stays within 1e-6 of its fp64 build on them
    (a tanh OUTPUT layer with one-hot targets is not: fp32 vs fp64 oracle differ by 1e-4..2e-2
    after 11 such steps, so it is not a parity case)."""
    p = synth.random_params(41, dims, 0.3)
    X, Y = synth.random_batch(42, 64, dims[0], dims[-1], "uniform")
    starts = list(range(0, 64, 6))          # 11 chained online steps
    net = make_net(dims, act, p)
    net.train_steps(dev(X), dev(Y), 1, starts, 0.1)
    ref, _ = oracle.Oracle(dims, act).train_steps(p, X, Y, 1, starts, 0.1)
    assert rel_err(gpu_params(net), ref) <= FP32_BAR


@pytest.mark.parametrize("dims,act,batch,steps", [
    ([784, 30, 10], "sigmoid", 1, 40),          # train_single on the c2 net
    ([200, 136, 72, 5], "tanh,sigmoid", 8, 10),  # no K6 for this net: one CTA up to ~1 M MAC/step
    ([3, 5, 2], "sigmoid", 8, 100),             # c1's shape
    ([100, 70, 40, 20, 3], "tanh,sigmoid", 5, 30),   # deeper net, thread-per-output layers
    ([64, 130, 9], "gaussian,sigmoid", 3, 25),  # warp-per-element delta (n_l >= 64)
    ([30, 40, 20, 8], "tanh,gaussian,sigmoid", 4, 20),   # one activation per layer
])
def test_small_batch_single_cta_path(dims, act, batch, steps):
    """nf_train_steps in the latency regime (a few rows per step, parameters in one SM's shared
    memory): the single-CTA kernel, parameters and per-step costs against the oracle."""
    p = synth.random_params(61 + batch, dims, 0.4)
    X, Y = synth.random_batch(62 + batch, 300, dims[0], dims[-1], "uniform")
    rng = np.random.default_rng(batch)
    starts = rng.integers(0, 300 - batch + 1, size=steps)
    net = make_net(dims, act, p)
    loss = torch.zeros(steps, device="cuda")
    n0 = nf.nf_launch_count()
    net.train_steps(dev(X), dev(Y), batch, starts, 0.5, step_loss=loss)
    assert nf.nf_launch_count() - n0 == 1          # one kernel for all steps
    ref, ref_loss = oracle.Oracle(dims, act).train_steps(p, X, Y, batch, starts, 0.5)
    assert rel_err(gpu_params(net), ref) <= FP32_BAR
    assert rel_err(loss.cpu().numpy(), ref_loss) <= FP32_BAR


def test_save_load_round_trip(tmp_path):
    """nf_save / nf_load: the loaded net has the same dims, activations and
    parameters bit for bit, and computes the same outputs."""
    dims, act = [37, 45, 20, 13], "tanh,gaussian,sigmoid"
    p = synth.random_params(81, dims, 0.5)
    net = make_net(dims, act, p)
    net.train_batch(dev(synth.random_batch(82, 64, 37, 13)[0]), dev(synth.random_batch(82, 64, 37, 13)[1]), 0.3)
    path = str(tmp_path / "net.txt")
    net.save(path)
    back = nf.Net.load(path)
    assert back.dims == dims and back.activation == act
    assert np.array_equal(gpu_params(back), gpu_params(net))
    x, _ = synth.random_batch(83, 50, 37, 13)
    assert np.array_equal(back.output(dev(x)).cpu().numpy(), net.output(dev(x)).cpu().numpy())


@pytest.mark.parametrize("dims,act,batch,steps", [
    ([784, 30, 10], "sigmoid", 1000, 45),        # K6; 20-step chunks of the staging pipeline
    ([200, 136, 72, 5], "tanh,sigmoid", 128, 7),  # generic kernels
])
def test_train_steps_from_host_dataset(dims, act, batch, steps):
    """nf_train_steps with the dataset in (pinned) host memory: each step's rows are copied in
    chunks overlapped with the training of the previous chunk; same result and per-step costs
    as the device-resident dataset (within the L2-reduction ordering of R12)."""
    p = synth.random_params(91, dims, 0.3)
    X, Y = synth.random_batch(92, 3 * batch, dims[0], dims[-1], "uniform")
    rng = np.random.default_rng(93)
    starts = rng.integers(0, 2 * batch + 1, size=steps)
    a, b = make_net(dims, act, p), make_net(dims, act, p)
    la, lb = torch.zeros(steps, device="cuda"), torch.zeros(steps, device="cuda")
    a.train_steps(torch.from_numpy(X).pin_memory(), torch.from_numpy(Y).pin_memory(), batch, starts, 0.5, step_loss=la)
    b.train_steps(dev(X), dev(Y), batch, starts, 0.5, step_loss=lb)
    assert rel_err(gpu_params(a), gpu_params(b)) <= 1e-5
    assert rel_err(la.cpu().numpy(), lb.cpu().numpy()) <= 1e-5
    ref, ref_loss = oracle.Oracle(dims, act).train_steps(p, X, Y, batch, starts, 0.5)
    assert rel_err(gpu_params(a), ref) <= FP32_BAR


@pytest.mark.parametrize("dims,act", [([20, 50, 5], "tanh,sigmoid"), ([784, 30, 10], "sigmoid")])
def test_eval_over_several_chunks(dims, act):
    """nf_output / nf_loss / nf_accuracy over 70,001 rows: more than two 32,768-row evaluation
    chunks with a ragged last one (generic K1 chain and the fused inference kernel); sampled
    outputs against the oracle, loss and accuracy against the oracle on all rows."""
    n = 70001
    p = synth.random_params(95, dims, 0.5)
    X, Y = synth.random_batch(96, n, dims[0], dims[-1], "uniform")
    net = make_net(dims, act, p)
    o = oracle.Oracle(dims, act)
    out = net.output(dev(X)).cpu().numpy()
    rows = np.r_[0:5, 32766:32771, 65534:65538, n - 5:n]
    assert rel_err(out[rows], o.output(p, np.ascontiguousarray(X[rows]))) <= FP32_BAR
    ref_loss = o.loss(p, X, Y)
    assert abs(net.loss(dev(X), dev(Y)) - ref_loss) <= FP32_BAR * ref_loss
    ref_out = o.output(p, X)
    mism, ties = argmax_agree(out, ref_out)
    assert mism == 0
    assert abs(net.accuracy(dev(X), dev(Y)) - o.accuracy(p, X, Y)) <= ties / n + 1e-6


@pytest.mark.parametrize("dims,act,batch", [([64, 256, 10], "tanh,sigmoid", 300), ([48, 1024, 7], "sigmoid", 520)])
def test_fused_output_layer_step_losses(dims, act, batch):
    """The per-step costs of nf_train_steps when the fused output-layer kernel computes them
    (per-block partials summed in fixed order by the tendency kernel) against the oracle."""
    p = synth.random_params(97, dims, 0.3)
    X, Y = synth.random_batch(98, 3 * batch, dims[0], dims[-1], "uniform")
    starts = [0, batch, 2 * batch, batch // 2, 7]
    net = make_net(dims, act, p)
    loss = torch.full((len(starts),), -1.0, device="cuda")
    net.train_steps(dev(X), dev(Y), batch, starts, 0.4, step_loss=loss)
    ref, ref_loss = oracle.Oracle(dims, act).train_steps(p, X, Y, batch, starts, 0.4)
    assert rel_err(loss.cpu().numpy(), ref_loss) <= FP32_BAR
    assert rel_err(gpu_params(net), ref) <= FP32_BAR


def test_save_load_fp64_keeps_the_doubles(tmp_path):
    """NF_MATH_FP64 nets save their double parameters (17 digits, never narrowed):
    save -> load -> save gives the identical file, the loaded net is in NF_MATH_FP64,
    and asking for an fp32 net from that file is rejected (NF_EFMT_PRECISION)."""
    dims, act = [37, 45, 13], "tanh,sigmoid"
    p = synth.random_params(84, dims, 0.5)
    net = make_net(dims, act, p)
    net.set_math(nf.NF_MATH_FP64)
    x, y = synth.random_batch(85, 64, 37, 13)
    net.train_batch(dev(x), dev(y), 0.3)      # doubles that are not fp32 values
    a, b = str(tmp_path / "a.net"), str(tmp_path / "b.net")
    net.save(a)
    text = open(a).read().split("\n")
    assert text[4] == "fp64"
    assert any(float(np.float32(float(v))) != float(v) for v in text[5:] if v)
    back = nf.Net.load(a)
    back.save(b)
    assert open(a).read() == open(b).read()
    assert np.array_equal(back.output(dev(x)).cpu().numpy(), net.output(dev(x)).cpu().numpy())
    with pytest.raises(nf.NFError) as e:
        nf.Net.load(a, math=nf.NF_MATH_FP32)
    assert e.value.code == nf.NF_EFMT_PRECISION


def test_deterministic_mode_is_bitwise_repeatable(tmp_path):
    """NF_SPLITK_DETERMINISTIC=1 (reading R12): two trainings from the same seed give
    bitwise-identical saved networks (SPEC acceptance 7) -- on the small-net path (the generic
    kernels replace K6, whose co_sum is an arrival-order L2 reduction) and on a wide net whose
    tensor-core steps use split-K and fused bias updates by default."""
    import subprocess
    import sys
    script = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import synth, paper_1902_06714_b200 as nf
out = sys.argv[2]
for tag, dims, act, B, math in [("c2", [784, 30, 10], "sigmoid", 1000, nf.NF_MATH_FP32),
                                ("wide", [784, 1024, 1024, 10], "tanh", 4096, nf.NF_MATH_TF32),
                                ("wide3", [784, 1024, 1024, 10], "tanh", 4096, nf.NF_MATH_FP32)]:
    X, Y = synth.random_batch(86, 3 * B, dims[0], dims[-1], "uniform")
    p = synth.random_params(87, dims, 0.05)
    for run in (0, 1):
        net = nf.Net(dims, act); net.set_math(math); net.set_params(torch.from_numpy(p).cuda())
        net.train_steps(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), B, [0, B, 2 * B, 7], 0.5)
        net.save(f"{out}/{tag}{run}.net")
'''
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, NF_SPLITK_DETERMINISTIC="1", NF_LOG_LAUNCHES="1")
    subprocess.run([sys.executable, "-c", script, root, str(tmp_path)], check=True, env=env, timeout=600)
    for tag in ("c2", "wide", "wide3"):
        assert open(tmp_path / f"{tag}0.net").read() == open(tmp_path / f"{tag}1.net").read(), tag
