"""Seeded synthetic inputs for the five BASELINE.json configs -- shared by the oracle
side (tests, bench cpu_baseline) and the CUDA side (tests, bench, smoke).

This module holds NONE of the method's arithmetic: it only draws random numbers
(numpy ``Generator(PCG64)``) and lays them out as fp32 arrays.  Every stream is
seeded ``SeedSequence([42, config_id, stream_id])`` with stream 0 = initial
parameters, 1 = x, 2 = labels, 3 = minibatch starts.

MNIST (the paper's dataset) is not in the container; these arrays
stand in for it with its shapes: 784 pixels in [0,1] with ~70 % exact zeros
(digit images are mostly background), and one-hot labels over 10 classes
(P:625-633).
"""
from __future__ import annotations

import numpy as np

# BASELINE.json "configs", in order (config_id = index + 1).
CONFIGS = {
    1: dict(name="c1-tiny", dims=[3, 5, 2], act="sigmoid", N=64, batch=8, steps=100, eta=1.0,
            init="unit", x="uniform", classes=2),
    2: dict(name="c2-digits-784-30-10", dims=[784, 30, 10], act="sigmoid", N=50000, batch=1000,
            steps=500, eta=3.0, init="xavier", x="digits", classes=10),
    3: dict(name="c3-wide-784-1024-1024-10", dims=[784, 1024, 1024, 10], act="tanh", N=200000,
            batch=4096, steps=240, eta=0.1, init="xavier", x="digits", classes=10),
    4: dict(name="c4-deep-784-256x8-10", dims=[784] + [256] * 8 + [10], act="relu,sigmoid",
            N=100000, batch=2048, steps=240, eta=0.05, init="he", x="digits", classes=10),
    5: dict(name="c5-large-4096x4-1024", dims=[4096, 4096, 4096, 4096, 1024], act="relu,sigmoid",
            N=131072, batch=16384, steps=50, eta=0.01, init="he", x="normal", classes=1024),
}


def _rng(config_id: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([42, config_id, stream])))


def init_params(config_id: int, dims=None, init: str | None = None) -> np.ndarray:
    """Flat fp32 parameters, for l = 1..L: W_l [n_l][n_{l-1}] row-major, then b_l [n_l].

    Draw order within stream 0: all of W_l (row-major), then b_l, layer by layer.
    W ~ N(0,1) * scale with scale = 1 ("unit"), 1/sqrt(fan_in) ("xavier") or
    sqrt(2/fan_in) ("he"), per BASELINE.json; b ~ N(0,1) (reading R2)."""
    cfg = CONFIGS[config_id]
    dims = cfg["dims"] if dims is None else list(dims)
    init = cfg["init"] if init is None else init
    rng = _rng(config_id, 0)
    out = []
    for l in range(1, len(dims)):
        fan_in = dims[l - 1]
        scale = {"unit": 1.0, "xavier": 1.0 / np.sqrt(fan_in), "he": np.sqrt(2.0 / fan_in)}[init]
        W = rng.standard_normal(dims[l] * fan_in) * scale
        b = rng.standard_normal(dims[l])
        out += [W, b]
    return np.concatenate(out).astype(np.float32)


def _x(config_id: int, kind: str, N: int, width: int) -> np.ndarray:
    rng = _rng(config_id, 1)
    X = np.empty((N, width), dtype=np.float32)
    chunk = max(1, (1 << 22) // width)
    for r0 in range(0, N, chunk):
        r1 = min(N, r0 + chunk)
        shape = (r1 - r0, width)
        if kind == "uniform":      # U[0,1)
            X[r0:r1] = rng.random(shape)
        elif kind == "digits":     # 0 w.p. 0.7, else U(0,1] drawn as 1 - U[0,1)
            keep = rng.random(shape) >= 0.7
            val = 1.0 - rng.random(shape)
            X[r0:r1] = np.where(keep, val, 0.0)
        elif kind == "normal":     # N(0,1)
            X[r0:r1] = rng.standard_normal(shape)
        else:
            raise ValueError(kind)
    return X


def labels(config_id: int, N: int | None = None) -> np.ndarray:
    cfg = CONFIGS[config_id]
    N = cfg["N"] if N is None else N
    return _rng(config_id, 2).integers(0, cfg["classes"], size=N).astype(np.int64)


def one_hot(lab: np.ndarray, classes: int) -> np.ndarray:
    Y = np.zeros((len(lab), classes), dtype=np.float32)
    Y[np.arange(len(lab)), lab] = 1.0
    return Y


def dataset(config_id: int, N: int | None = None):
    """(X [N][n_0] fp32, Y [N][n_L] fp32 one-hot).  N defaults to the config's."""
    cfg = CONFIGS[config_id]
    N = cfg["N"] if N is None else N
    X = _x(config_id, cfg["x"], N, cfg["dims"][0])
    Y = one_hot(labels(config_id, N), cfg["classes"])
    return X, Y


def batch_starts(config_id: int, steps: int | None = None, N: int | None = None,
                 batch: int | None = None) -> np.ndarray:
    """0-based minibatch starts uniform in [0, N - batch] (reading R11)."""
    cfg = CONFIGS[config_id]
    steps = cfg["steps"] if steps is None else steps
    N = cfg["N"] if N is None else N
    batch = cfg["batch"] if batch is None else batch
    return _rng(config_id, 3).integers(0, N - batch + 1, size=steps).astype(np.int64)


# -- generic helpers for property tests (random small nets) ------------------
def random_params(seed: int, dims, scale: float = 1.0) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([7, seed])))
    n = sum(dims[l] * dims[l - 1] + dims[l] for l in range(1, len(dims)))
    return (rng.standard_normal(n) * scale).astype(np.float32)


def random_batch(seed: int, n: int, n_in: int, n_out: int, x_kind: str = "uniform"):
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([9, seed])))
    if x_kind == "uniform":
        x = rng.random((n, n_in))
    elif x_kind == "normal":
        x = rng.standard_normal((n, n_in))
    else:
        raise ValueError(x_kind)
    lab = rng.integers(0, n_out, size=n)
    return x.astype(np.float32), one_hot(lab, n_out)
