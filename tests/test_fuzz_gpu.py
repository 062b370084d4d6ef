"""Seeded random sweep over the dispatch space (-m gpu): depth, widths (ragged, 1..300),
one activation per layer, batch (1..700: the single-CTA, K6, fused output-layer, tensor-core
and SIMT paths), numerics mode and entry point, each against the fp64 oracle.  Catches
dispatch-boundary bugs the hand-picked shapes miss."""
import numpy as np
import pytest
import torch

import oracle
import synth
from parity import FP32_BAR, FP64_BAR, TF32_BAR, rel_err

pytestmark = pytest.mark.gpu

import paper_1902_06714_b200 as nf  # noqa: E402

SMOOTH = ["sigmoid", "tanh", "gaussian"]   # no kinks (relu / step are covered elsewhere, R8)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def case(seed):
    rng = np.random.default_rng(1000 + seed)
    L = int(rng.integers(1, 5))
    widths = [int(rng.choice([rng.integers(1, 40), rng.integers(40, 300)])) for _ in range(L + 1)]
    acts = ",".join(rng.choice(SMOOTH, size=L))
    batch = int(rng.choice([1, 2, 7, 64, 257, 700]))
    math = int(rng.choice([nf.NF_MATH_FP32, nf.NF_MATH_FP32, nf.NF_MATH_TF32, nf.NF_MATH_FP64]))
    api = str(rng.choice(["steps_dev", "steps_host", "batch", "grad", "output"]))
    return widths, acts, batch, math, api


def check(got, ref, math, ref32=None):
    """fp64 mode: FP64_BAR.  fp32 mode: FP32_BAR, or 10x the deviation of the oracle's own fp32
    build from its fp64 build when a random net is ill-conditioned (a 1-wide tanh bottleneck
    turns fp32 rounding into 5e-3 after four steps: arithmetic, not a bug; the kernels' SFU
    exp (2^-21 relative) adds to the libm-exact oracle where errors grow 4x per step).  TF32 tiles:
    TF32_BAR normwise (R14b), or for an ill-conditioned net the fp32 oracle's deviation scaled by
    the ratio of the two unit roundoffs (2^-11 / 2^-24), whichever is larger."""
    if math == nf.NF_MATH_FP64:
        assert rel_err(got, ref) <= FP64_BAR
    elif math == nf.NF_MATH_FP32:
        bar = FP32_BAR if ref32 is None else max(FP32_BAR, 10 * rel_err(ref32, ref))
        assert rel_err(got, ref) <= bar
    else:
        bar = TF32_BAR if ref32 is None else max(TF32_BAR, 2.0 ** 13 * rel_err(ref32, ref, tau=1.0))
        assert rel_err(got, ref, tau=1.0) <= bar


@pytest.mark.parametrize("seed", range(200))
def test_random_case(seed):
    dims, acts, batch, math, api = case(seed)
    p = synth.random_params(2000 + seed, dims, 0.5).astype(np.float32).astype(np.float64)
    N = 3 * batch + 5
    X, Y = synth.random_batch(3000 + seed, N, dims[0], dims[-1], "uniform")
    net = nf.Net(dims, acts)
    net.set_params(dev(p.astype(np.float32)))
    net.set_math(math)
    o = oracle.Oracle(dims, acts)
    o32 = oracle.Oracle(dims, acts, bits=32)
    eta = float(np.float32(0.3))
    if api in ("steps_dev", "steps_host"):
        starts = np.random.default_rng(seed).integers(0, N - batch + 1, size=4)
        Xs = dev(X) if api == "steps_dev" else torch.from_numpy(X).pin_memory()
        Ys = dev(Y) if api == "steps_dev" else torch.from_numpy(Y).pin_memory()
        net.train_steps(Xs, Ys, batch, starts, eta)
        got = net.get_params()
        ref, _ = o.train_steps(p, X, Y, batch, starts, eta)
        ref32, _ = o32.train_steps(p.astype(np.float32), X, Y, batch, starts, eta)
        check(got, ref, math, ref32)
    elif api == "batch":
        net.train_batch(dev(X[:batch]), dev(Y[:batch]), eta)
        ref, _ = o.train_batch(p, X[:batch], Y[:batch], eta)
        ref32, _ = o32.train_batch(p.astype(np.float32), X[:batch], Y[:batch], eta)
        check(net.get_params(), ref, math, ref32)
    elif api == "grad":
        g = net.grad(dev(X[:batch]), dev(Y[:batch])).cpu().numpy()
        check(g, o.grad(p, X[:batch], Y[:batch]), math, o32.grad(p.astype(np.float32), X[:batch], Y[:batch]))
    else:
        out = net.output(dev(X[:batch])).cpu().numpy()
        check(out, o.output(p, X[:batch]), math, o32.output(p.astype(np.float32), X[:batch]))
