"""Pins of the batched fp64 oracle (oracle/batched.py) -- -m "not gpu".

The batched oracle is the definition of one SGD step written over a whole batch with numpy's
fp64 matrix product as the contraction; it exists because the per-sample C
oracle cannot reach the bench sizes.  It is pinned to things other than itself:
  * the independently pinned C oracle (tests/test_oracle.py: closed forms, FD, golden values)
    on random nets of every activation, every output it produces (1e-12 relative: the two
    differ only in the summation order inside the products);
  * the closed-form single sigmoid neuron;
  * centered finite differences of its own cost (fp64, h = 1e-6);
  * the co_sum split identity and eta = 0 / duplicate-batch invariances.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle.batched import BatchedOracle

ACTS = ["sigmoid", "tanh", "relu", "gaussian", "step", "relu,sigmoid", "tanh,gaussian,sigmoid"]


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("act", ACTS)
def test_equals_c_oracle(act):
    dims = [7, 9, 6, 4] if act != "tanh,gaussian,sigmoid" else [7, 9, 6, 4]
    p = synth.random_params(11, dims, 0.8)
    x, y = synth.random_batch(12, 37, dims[0], dims[-1], "normal")
    c, b = oracle.Oracle(dims, act), BatchedOracle(dims, act)
    assert _rel(b.output(p, x), c.output(p, x)) <= 1e-12
    assert _rel(b.grad(p, x, y), c.grad(p, x, y)) <= 1e-12
    pb, lb, _ = b.train_batch(p, x, y, 0.7)
    pc, lc = c.train_batch(p, x, y, 0.7)
    assert _rel(pb, pc) <= 1e-12 and abs(lb - lc) <= 1e-12 * abs(lc)
    assert abs(b.loss(p, x, y) - c.loss(p, x, y)) <= 1e-12 * c.loss(p, x, y)
    assert b.accuracy(p, x, y) == c.accuracy(p, x, y)
    A, Z = b.forward(p, x)
    As, Ds = c.stash(p, x, y)
    D = b.backward(p, A, Z, y)
    for l in range(1, len(dims)):
        assert _rel(A[l], As[l]) <= 1e-12
        assert _rel(D[l], Ds[l - 1]) <= 1e-12


def test_single_sigmoid_neuron_closed_form():
    """dims [n,1], sigmoid: dC/dw = (a-y) a (1-a) x, dC/db = (a-y) a (1-a); w = 0, b = 0, y = 1
    gives a = 1/2 and delta = -1/8 exactly."""
    o = BatchedOracle([3, 1], "sigmoid")
    x = np.array([[0.5, -2.0, 4.0]], np.float32)
    G = o.grad(np.zeros(4), x, np.array([[1.0]], np.float32))
    assert np.array_equal(G, np.array([-0.0625, 0.25, -0.5, -0.125]))
    rng = np.random.default_rng(3)
    w, b = rng.standard_normal(3), 0.3
    a = 1 / (1 + np.exp(-(x[0].astype(np.float64) @ w + b)))
    G = o.grad(np.concatenate([w, [b]]), x, np.array([[0.2]], np.float32))
    d = (a - float(np.float32(0.2))) * a * (1 - a)   # y is an fp32 value widened exactly
    assert np.allclose(G, np.concatenate([d * x[0], [d]]), rtol=1e-12, atol=0)


@pytest.mark.parametrize("act", ["sigmoid", "tanh", "gaussian", "tanh,gaussian,sigmoid"])
def test_grad_matches_centered_fd(act):
    dims = [4, 6, 5, 3]
    o = BatchedOracle(dims, act)
    p = synth.random_params(21, dims, 0.8).astype(np.float64)
    x, y = synth.random_batch(22, 5, dims[0], dims[-1], "normal")
    G = o.grad(p, x, y)
    h, n = 1e-6, x.shape[0]
    scale = np.abs(G).max()
    for i in range(p.size):
        q = p.copy(); q[i] += h; cp = o.loss(q, x, y) * n
        q[i] -= 2 * h; cm = o.loss(q, x, y) * n
        fd = (cp - cm) / (2 * h)
        assert abs(fd - G[i]) <= 1e-5 * max(abs(G[i]), 1e-3 * scale), (act, i, fd, G[i])


def test_relu_all_active_is_linear_least_squares():
    """relu with every pre-activation > 0 is linear: dC/dW = sum_s (W x_s + b - y_s) x_s^T."""
    o = BatchedOracle([4, 3], "relu")
    rng = np.random.default_rng(5)
    W = rng.uniform(0.5, 1.0, (3, 4)); b = np.full(3, 0.5)
    x = rng.uniform(0.1, 1.0, (6, 4)).astype(np.float32)
    y = rng.uniform(0, 1, (6, 3)).astype(np.float32)
    G = o.grad(np.concatenate([W.ravel(), b]), x, y)
    r = x.astype(np.float64) @ W.T + b - y
    assert np.allclose(G, np.concatenate([(r.T @ x).ravel(), r.sum(0)]), rtol=1e-13, atol=1e-13)


def test_co_sum_split_identity_and_invariances():
    """G(batch) = G(part1) + G(part2); eta = 0 leaves params unchanged;
    a duplicated batch gives the same update under eta/B."""
    dims = [8, 7, 5]
    o = BatchedOracle(dims, "tanh")
    p = synth.random_params(31, dims, 0.6)
    x, y = synth.random_batch(32, 40, 8, 5, "uniform")
    G = o.grad(p, x, y)
    for k in (1, 13, 39):
        assert np.allclose(G, o.grad(p, x[:k], y[:k]) + o.grad(p, x[k:], y[k:]), rtol=1e-12, atol=1e-14)
    q, _, _ = o.train_batch(p, x, y, 0.0)
    assert np.array_equal(q, p.astype(np.float64))
    q1, _, _ = o.train_batch(p, x, y, 0.9)
    q2, _, _ = o.train_batch(p, np.concatenate([x, x]), np.concatenate([y, y]), 0.9)
    assert np.allclose(q1, q2, rtol=1e-14, atol=1e-15)


def test_kink_free_rows_and_decision_override():
    """zdec only moves relu/step decisions: with zdec = Z the result is unchanged; rows with a
    pre-activation inside the margin band are dropped."""
    dims = [5, 6, 3]
    o = BatchedOracle(dims, "relu,sigmoid")
    p = synth.random_params(41, dims, 0.9)
    x, y = synth.random_batch(42, 20, 5, 3, "normal")
    A, Z = o.forward(p, x)
    assert np.array_equal(o.grad(p, x, y), o.grad(p, x, y, zdec=Z))
    ok = o.kink_free_rows(Z, 0.05)
    rms = np.sqrt(np.mean(Z[1] ** 2))
    assert np.array_equal(ok, np.all(np.abs(Z[1]) > 0.05 * rms, axis=1))
    # forcing a decision flips exactly that unit's delta
    zd = [None] + [z.copy() for z in Z[1:]]
    zd[1][0, 0] = -zd[1][0, 0] if zd[1][0, 0] != 0 else 1.0
    D0 = o.backward(p, A, Z, y)
    D1 = o.backward(p, A, Z, y, zdec=zd)
    diff = np.argwhere(D0[1] != D1[1])
    assert diff.tolist() in ([[0, 0]], [])
