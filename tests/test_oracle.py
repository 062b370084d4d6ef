"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the passage it follows ("P:n" = PAPER.md line, "S:n" = SPEC.md line).
None of these compares the oracle with itself: the expected values are closed
forms, printed values (tests/golden/), finite differences, algebraic identities
of the batch sum, or brute force on tiny inputs.
"""
import math
import os

import numpy as np
import pytest

import oracle
import synth

O64 = lambda dims, act="sigmoid": oracle.Oracle(dims, act, bits=64)  # noqa: E731


def _read_golden(golden_dir, name):
    rows = []
    for line in open(os.path.join(golden_dir, name)):
        line = line.split("#", 1)[0].strip()
        if line:
            rows.append(line.split())
    return rows


# --------------------------------------------------------------------------- activations
def test_activation_golden(golden_dir):
    o = O64([1, 1])
    for fn, kind, x, exp, tol in _read_golden(golden_dir, "activations.txt"):
        got = o.act(kind, float(x)) if fn == "act" else o.act_prime(kind, float(x))
        assert abs(got - float(exp)) <= float(tol), (fn, kind, x, got, exp)


@pytest.mark.parametrize("kind", ["sigmoid", "tanh", "relu", "gaussian"])
def test_activation_prime_matches_centered_fd(kind):
    """sigma' equals a centered FD of sigma (h=1e-6) to 1e-6 relative, 100 points in [-5,5]."""
    o = O64([1, 1])
    rng = np.random.default_rng(1)
    xs = rng.uniform(-5, 5, 100)
    h = 1e-6
    for x in xs:
        if kind == "relu" and abs(x) < 1e-3:
            continue
        fd = (o.act(kind, x + h) - o.act(kind, x - h)) / (2 * h)
        d = o.act_prime(kind, x)
        assert abs(fd - d) <= 1e-6 * max(abs(d), 1e-3), (kind, x, fd, d)


def test_activation_ranges():
    """sigmoid in (0,1), tanh in (-1,1), relu >= 0, step in {0,1}, gaussian in (0,1]."""
    o = O64([1, 1])
    for x in np.linspace(-30, 30, 121):
        assert 0 < o.act("sigmoid", x) < 1 or abs(x) > 30
        assert -1 <= o.act("tanh", x) <= 1
        assert o.act("relu", x) >= 0
        assert o.act("step", x) in (0.0, 1.0)
        assert 0 <= o.act("gaussian", x) <= 1


def test_unknown_activation_is_an_error():
    """an unknown name is an error, never a silent default."""
    with pytest.raises(ValueError):
        O64([2, 2], "softmax")
    with pytest.raises(ValueError):
        O64([2], "sigmoid")          # dims=[2] -> construction error
    with pytest.raises(ValueError):
        O64([2, 0, 1], "sigmoid")    # every dim >= 1


def test_activation_spec_forms():
    """One name -> every layer; "hidden,output" -> hidden / output (R7); L names -> one per
    layer; any other count is an error."""
    A = oracle.ACT
    assert oracle.parse_activation("tanh", 3) == [A["tanh"]] * 3
    assert oracle.parse_activation("relu,sigmoid", 4) == [A["relu"]] * 3 + [A["sigmoid"]]
    assert oracle.parse_activation("relu,tanh,gaussian", 3) == [A["relu"], A["tanh"], A["gaussian"]]
    assert oracle.parse_activation("relu,sigmoid", 1) == [A["sigmoid"]]
    with pytest.raises(ValueError):
        oracle.parse_activation("relu,tanh,sigmoid", 4)
    with pytest.raises(ValueError):
        O64([2, 3, 4, 2], "relu,tanh,sigmoid,step")


def test_per_layer_activations_reduce_to_the_shared_forms():
    """A per-layer list with the hidden name repeated is the "hidden,output" net, bit for bit;
    a list of one name is the single-name net."""
    dims = [5, 7, 6, 3]
    p = synth.random_params(3, dims, 0.7).astype(np.float64)
    x, y = synth.random_batch(4, 9, 5, 3, "normal")
    assert np.array_equal(O64(dims, "tanh,tanh,sigmoid").grad(p, x, y), O64(dims, "tanh,sigmoid").grad(p, x, y))
    assert np.array_equal(O64(dims, "gaussian,gaussian,gaussian").output(p, x), O64(dims, "gaussian").output(p, x))
    # and the order matters: swapping two hidden activations changes the output
    assert not np.array_equal(O64(dims, "tanh,gaussian,sigmoid").output(p, x),
                              O64(dims, "gaussian,tanh,sigmoid").output(p, x))


@pytest.mark.parametrize("acts", ["tanh,gaussian,sigmoid,tanh", "sigmoid,tanh,gaussian,sigmoid"])
def test_per_layer_backprop_matches_centered_fd(acts):
    """Backprop with a different activation in every layer: every dW, db entry equals the
    centered FD (h = 1e-6) of the cost (fp64, rel 1e-5) -- the per-layer sigma' indexing."""
    dims = [4, 6, 5, 3, 2]
    o = O64(dims, acts)
    p = synth.random_params(77, dims, 0.8).astype(np.float64)
    x, y = synth.random_batch(78, 3, dims[0], dims[-1], "normal")
    G = o.grad(p, x, y)
    h = 1e-6
    scale = max(np.abs(G).max(), 1e-8)
    for i in range(p.size):
        q = p.copy(); q[i] += h; cp = o.loss(q, x, y) * 3
        q[i] -= 2 * h; cm = o.loss(q, x, y) * 3
        fd = (cp - cm) / (2 * h)
        assert abs(fd - G[i]) <= 1e-5 * max(abs(G[i]), 1e-3 * scale), (acts, i, fd, G[i])


# --------------------------------------------------------------------------- shapes
def test_param_counts(golden_dir):
    g = {k: float(v) for k, v in _read_golden(golden_dir, "paper_numbers.txt")}
    assert O64([3, 5, 2]).n_params == g["param_count_3_5_2"]
    assert O64([784, 30, 10]).n_params == g["param_count_784_30_10"]
    assert 50000 // 1000 == g["mnist_batches_per_epoch_b1000"]


# --------------------------------------------------------------------------- forward
def test_forward_spec_examples():
    # S:133 / S:143: all-zero weights and biases, sigmoid, dims [2,1] -> 0.5
    o = O64([2, 1], "sigmoid")
    out = o.output(np.zeros(3), np.array([[7, -7]], np.float32))
    assert out[0, 0] == 0.5
    # dims [1,1], W=2, b=-1, relu, x=3 -> z = 5, a = 5
    o = O64([1, 1], "relu")
    assert o.output(np.array([2.0, -1.0]), np.array([[3]], np.float32))[0, 0] == 5.0


def _np_forward(dims, acts, params, x):
    """Eq. 2 with numpy matmul as the contraction (brute-force cross-check)."""
    f = {"sigmoid": lambda z: 1 / (1 + np.exp(-z)), "tanh": np.tanh,
         "relu": lambda z: np.maximum(z, 0), "gaussian": lambda z: np.exp(-z * z),
         "step": lambda z: (z > 0).astype(np.float64)}
    a, o = x.astype(np.float64), 0
    L = len(dims) - 1
    for l in range(1, L + 1):
        W = params[o:o + dims[l] * dims[l - 1]].reshape(dims[l], dims[l - 1]); o += W.size
        b = params[o:o + dims[l]]; o += dims[l]
        a = f[acts[0] if l < L else acts[1]](a @ W.T + b)
    return a


@pytest.mark.parametrize("seed", range(6))
def test_output_matches_matmul_forward(seed):
    rng = np.random.default_rng(seed)
    dims = list(rng.integers(1, 9, size=rng.integers(2, 6)))
    acts = [("sigmoid", "sigmoid"), ("tanh", "tanh"), ("relu", "sigmoid"), ("gaussian", "gaussian"),
            ("step", "sigmoid"), ("relu", "relu")][seed]
    p = synth.random_params(seed, dims).astype(np.float64)
    x, _ = synth.random_batch(seed, 5, dims[0], dims[-1], "normal")
    o = O64(dims, ",".join(acts))
    np.testing.assert_allclose(o.output(p, x), _np_forward(dims, acts, p, x), rtol=1e-12, atol=1e-14)


def test_output_equals_cached_forward_bitwise():
    """S:144 / S:209: output(net, x) == a_L after fwdprop(net, x), bitwise."""
    dims = [4, 5, 3]
    o = O64(dims, "tanh")
    p = synth.random_params(3, dims).astype(np.float64)
    x, y = synth.random_batch(3, 6, 4, 3)
    A, _ = o.stash(p, x, y)
    assert np.array_equal(o.output(p, x), A[-1])
    assert np.array_equal(A[0], x.astype(np.float64))


# --------------------------------------------------------------------------- backprop
def test_single_sigmoid_neuron_exact():
    """dims [n,1], w=0, b=0, y=1: a=1/2, delta=(1/2-1)*1/4=-1/8 (P:111 quadratic cost,
    P:207-209 sigmoid); dC/dw = -x/8, dC/db = -1/8 -- all exactly representable."""
    n = 5
    o = O64([n, 1], "sigmoid")
    x = np.array([[0.5, 1.0, -2.0, 0.25, 3.0]], np.float32)
    G = o.grad(np.zeros(n + 1), x, np.ones((1, 1), np.float32))
    assert np.array_equal(G[:n], -x[0].astype(np.float64) / 8)
    assert G[n] == -0.125


@pytest.mark.parametrize("seed", range(4))
def test_single_sigmoid_neuron_closed_form(seed):
    """Closed form of one sigmoid neuron: dC/dw = (a-y) a (1-a) x, dC/db = (a-y) a (1-a)."""
    rng = np.random.default_rng(seed)
    n = 7
    w, b = rng.standard_normal(n), rng.standard_normal()
    x = rng.standard_normal((1, n)).astype(np.float32)
    y = np.float32(rng.random())
    a = 1 / (1 + math.exp(-(float(np.dot(w, x[0].astype(np.float64))) + b)))
    dz = (a - float(y)) * a * (1 - a)
    G = O64([n, 1]).grad(np.concatenate([w, [b]]), x, np.array([[y]], np.float32))
    np.testing.assert_allclose(G[:n], dz * x[0].astype(np.float64), rtol=1e-12)
    np.testing.assert_allclose(G[n], dz, rtol=1e-12)


def test_relu_all_active_is_linear_least_squares():
    """With every relu active the layer is affine; the gradient of
    1/2 sum_s ||W x_s + b - y_s||^2 is sum_s (W x_s + b - y_s) x_s^T (textbook LS)."""
    rng = np.random.default_rng(5)
    ni, no, n = 6, 4, 9
    W = rng.uniform(0.1, 1.0, (no, ni)); b = rng.uniform(0.1, 1.0, no)
    x = rng.uniform(0.1, 1.0, (n, ni)).astype(np.float32)
    y = rng.uniform(0, 1, (n, no)).astype(np.float32)
    G = O64([ni, no], "relu").grad(np.concatenate([W.ravel(), b]), x, y)
    xd = x.astype(np.float64)
    R = xd @ W.T + b - y
    np.testing.assert_allclose(G[:no * ni].reshape(no, ni), R.T @ xd, rtol=1e-12)
    np.testing.assert_allclose(G[no * ni:], R.sum(0), rtol=1e-12)


def test_exact_fit_gives_zero_tendency():
    """dims [1,1], sigmoid, w=0, b=0, x=0, y=0.5 -> all tendencies zero."""
    G = O64([1, 1]).grad(np.zeros(2), np.zeros((1, 1), np.float32), np.full((1, 1), 0.5, np.float32))
    assert np.all(G == 0)


FD_ACTS = ["sigmoid", "tanh", "gaussian", "relu,sigmoid", "tanh,relu"]


@pytest.mark.parametrize("seed", range(25))
def test_backprop_matches_centered_fd(seed):
    """S:154 / S:210 / S:527: every dW, db entry equals the centered FD (h=1e-6) of the
    quadratic cost C = sum_s 1/2 ||a_L(x_s) - y_s||^2 to rel 1e-5 (fp64)."""
    rng = np.random.default_rng(100 + seed)
    dims = [int(v) for v in rng.integers(1, 9, size=rng.integers(2, 6))]
    act = FD_ACTS[seed % len(FD_ACTS)]
    o = O64(dims, act)
    p = synth.random_params(100 + seed, dims, 0.8).astype(np.float64)
    n = 3
    x, y = synth.random_batch(100 + seed, n, dims[0], dims[-1], "normal")
    G = o.grad(p, x, y)
    h = 1e-6
    C = lambda q: o.loss(q, x, y) * n  # noqa: E731  (orc_loss is the mean, reading R9)
    scale = max(np.abs(G).max(), 1e-8)
    for i in range(p.size):
        q = p.copy(); q[i] += h; cp = C(q)
        q[i] -= 2 * h; cm = C(q)
        fd = (cp - cm) / (2 * h)
        if "relu" in act and abs(fd - G[i]) > 1e-5 * max(abs(G[i]), 1e-3 * scale):
            # a relu kink inside [p-h, p+h] makes the FD meaningless; skip that entry
            A, _ = o.stash(q + h, x, y)
            if any(np.min(np.abs(a)) < 1e-5 for a in A[1:-1]):
                continue
        assert abs(fd - G[i]) <= 1e-5 * max(abs(G[i]), 1e-3 * scale), (dims, act, i, fd, G[i])


# --------------------------------------------------------------------------- batch sum (co_sum)
@pytest.mark.parametrize("split", [1, 3, 7, 12])
def test_batch_sum_split_invariance(split):
    """P:511-516, P:536-556 (co_sum): the tendency of a batch is the sum of the tendencies
    of any split of it."""
    dims = [6, 5, 4]
    o = O64(dims, "tanh")
    p = synth.random_params(11, dims).astype(np.float64)
    x, y = synth.random_batch(11, 13, 6, 4)
    G = o.grad(p, x, y)
    G2 = o.grad(p, x[:split], y[:split]) + o.grad(p, x[split:], y[split:])
    np.testing.assert_allclose(G, G2, rtol=1e-12, atol=1e-14)


def test_batch_sum_equals_per_sample_sum_exactly():
    """B=4 on dims [3,4,2]: batch tendency == sum of 4 single-sample tendencies
    summed in column order (same additions in the same order -> bitwise)."""
    dims = [3, 4, 2]
    o = O64(dims)
    p = synth.random_params(2, dims).astype(np.float64)
    x, y = synth.random_batch(2, 4, 3, 2)
    acc = np.zeros(o.n_params)
    for s in range(4):
        acc = acc + o.grad(p, x[s:s + 1], y[s:s + 1])
    assert np.array_equal(o.grad(p, x, y), acc)


def test_duplicate_batch_invariance():
    """duplicating every sample leaves the eta/B-scaled update unchanged."""
    dims = [5, 6, 3]
    o = O64(dims)
    p = synth.random_params(4, dims).astype(np.float64)
    x, y = synth.random_batch(4, 7, 5, 3)
    p1, _ = o.train_batch(p, x, y, 0.5)
    p2, _ = o.train_batch(p, np.concatenate([x, x]), np.concatenate([y, y]), 0.5)
    np.testing.assert_allclose(p1, p2, rtol=1e-13, atol=1e-15)


def test_batch_of_one_is_train_single():
    """S:175 / S:183: train_batch with one column == fwdprop, backprop, update(eta)."""
    dims = [4, 3, 2]
    o = O64(dims)
    p = synth.random_params(8, dims).astype(np.float64)
    x, y = synth.random_batch(8, 1, 4, 2)
    p1, _ = o.train_batch(p, x, y, 0.3)
    assert np.array_equal(p1, p - 0.3 * o.grad(p, x, y))


# --------------------------------------------------------------------------- update
def test_eta_zero_is_bitwise_noop():
    """S:163 / S:174."""
    dims = [4, 5, 3]
    o = O64(dims)
    p = synth.random_params(9, dims).astype(np.float64)
    x, y = synth.random_batch(9, 5, 4, 3)
    p1, _ = o.train_batch(p, x, y, 0.0)
    assert np.array_equal(p1, p)


def test_update_scale_is_eta_over_batch():
    """Reading R3: W -= (eta/B) * sum of tendencies."""
    dims = [4, 5, 3]
    o = O64(dims)
    p = synth.random_params(10, dims).astype(np.float64)
    x, y = synth.random_batch(10, 6, 4, 3)
    p1, _ = o.train_batch(p, x, y, 1.2)
    np.testing.assert_allclose(p1, p - (1.2 / 6) * o.grad(p, x, y), rtol=1e-15, atol=1e-16)


def test_descent_at_small_eta():
    """a small step along the negative gradient lowers the batch cost."""
    for seed in range(5):
        dims = [5, 6, 3]
        o = O64(dims, ["sigmoid", "tanh", "relu,sigmoid", "gaussian", "tanh"][seed])
        p = synth.random_params(20 + seed, dims).astype(np.float64)
        x, y = synth.random_batch(20 + seed, 8, 5, 3)
        before = o.loss(p, x, y)
        p1, l0 = o.train_batch(p, x, y, 0.01)
        assert l0 == pytest.approx(before, rel=1e-15)
        assert o.loss(p1, x, y) < before


def test_train_steps_is_the_minibatch_loop():
    """epochs x minibatches, each a train call on a contiguous slice."""
    dims = [3, 5, 2]
    o = O64(dims)
    p = synth.init_params(1)
    X, Y = synth.dataset(1)
    starts = synth.batch_starts(1, steps=10)
    pa, la = o.train_steps(p, X, Y, 8, starts, 1.0)
    q = p.astype(np.float64)
    for i, s in enumerate(starts):
        q, l = o.train_batch(q, X[s:s + 8], Y[s:s + 8], 1.0)
        assert l == la[i]
    assert np.array_equal(pa, q)


# --------------------------------------------------------------------------- loss / accuracy
def test_loss_pins():
    # output equals y exactly -> 0 (zero sigmoid net outputs 1/2)
    o = O64([3, 2])
    x = np.ones((4, 3), np.float32)
    assert o.loss(np.zeros(8), x, np.full((4, 2), 0.5, np.float32)) == 0.0
    # forced output 1 (relu, w=0, b=1), y=0 -> 1/2 * 1^2 = 0.5
    o = O64([1, 1], "relu")
    assert o.loss(np.array([0.0, 1.0]), np.zeros((3, 1), np.float32), np.zeros((3, 1), np.float32)) == 0.5


def test_accuracy_pins():
    # output forced to the one-hot of the label -> 1.0  (relu identity net, x = y)
    k = 5
    o = O64([k, k], "relu")
    p = np.concatenate([np.eye(k).ravel(), np.zeros(k)])
    lab = np.array([0, 3, 4, 1, 1, 2, 0])
    Y = synth.one_hot(lab, k)
    assert o.accuracy(p, Y, Y) == 1.0
    # predicting class (label+1) mod k everywhere -> 0.0
    P = np.roll(np.eye(k), 1, axis=0)
    assert o.accuracy(np.concatenate([P.ravel(), np.zeros(k)]), Y, Y) == 0.0
    # n = 0 -> 0.0
    assert o.accuracy(p, np.zeros((0, k), np.float32), np.zeros((0, k), np.float32)) == 0.0
    # ties -> lowest index: zero net -> all outputs equal -> predicts class 0
    z = np.zeros(k * k + k)
    assert o.accuracy(z, Y, Y) == pytest.approx(np.mean(lab == 0))


def test_untrained_c2_accuracy_is_chance(golden_dir):
    """P:754 / P:766-771: an untrained 784-30-10 net predicts at chance (~10 %)."""
    g = {k: float(v) for k, v in _read_golden(golden_dir, "paper_numbers.txt")}
    o = O64([784, 30, 10])
    X, Y = synth.dataset(2, N=2000)
    acc = o.accuracy(synth.init_params(2), X, Y)
    assert abs(acc - g["initial_accuracy_pct"] / 100) < 0.05


# --------------------------------------------------------------------------- precision builds
def test_real32_build_tracks_real64():
    """The real32 build (P:253-256 default precision) agrees with real64 to fp32 rounding."""
    dims = [784, 30, 10]
    p = synth.init_params(2)
    X, Y = synth.dataset(2, N=64)
    g64 = oracle.Oracle(dims, bits=64).grad(p, X, Y)
    g32 = oracle.Oracle(dims, bits=32).grad(p, X, Y)
    assert np.max(np.abs(g32 - g64)) <= 1e-4 * np.max(np.abs(g64))


def test_per_layer_forward_matches_numpy_closed_forms():
    """Per-layer activations against numpy's own closed forms (tanh, e^{-z^2}, 1/(1+e^{-z})):
    layer l uses the l-th name."""
    dims = [3, 4, 5, 2]
    p = synth.random_params(5, dims, 0.9).astype(np.float64)
    x, _ = synth.random_batch(6, 7, 3, 2, "normal")
    o = O64(dims, "tanh,gaussian,sigmoid")
    (W1, b1), (W2, b2), (W3, b3) = o.layers(p)
    a = np.tanh(x.astype(np.float64) @ W1.T + b1)
    a = np.exp(-(a @ W2.T + b2) ** 2)
    a = 1.0 / (1.0 + np.exp(-(a @ W3.T + b3)))
    np.testing.assert_allclose(o.output(p, x), a, rtol=1e-12, atol=1e-14)
