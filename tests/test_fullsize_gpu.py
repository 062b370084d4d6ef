"""Full-size training steps against the batched fp64 oracle, in the launch configuration bench.py
times (-m gpu).

Each case runs ONE SGD step through ``nf_train_steps`` -- the call bench.py times, so the same
CUDA-graph-captured kernel sequence, tile shapes, split-K and epilogue variants (the SGD
update epilogues with their split-K L2 reductions, the fused bias updates, the persistent
1xTF32 kernels) -- at the configuration's batch size, and compares it with one
``train_batch`` step of ``oracle/batched.py``:

  * the applied update W' - W and b' - b of every layer (the batch-summed tendencies times
    eta/B) at the north-star bars: 1e-4 (tau = 0.1) in NF_MATH_FP32, 5e-3 normwise
    (tau = 1) in NF_MATH_TF32 (reading R14b);
  * the step's mean cost (R9).

The update is compared, not W' itself: W' = W - update would hide the tendency's error behind
W.  Its fp32 storage rounds: each in-place add to W (the SGD epilogue, or one per split-K term /
bias strip reduced in L2) costs at most 1/2 ulp of W', so the allowance is that many half-ulps
on top of the relative bar; eta is raised so the update is a sizeable fraction of W (the
step is linear in eta) and those ulps stay far below the bar.

Relu decisions (reading R8): rows whose fp64 pre-activations fall inside a band around the kink
where an fp32 / TF32 sum may decide relu' differently are not used -- the batch is drawn from
a larger seeded pool of the config's inputs, keeping kink-free rows.  At config 5's widths no
row is kink-free at the TF32 band, so TF32 is checked there on the same shapes with a smooth
hidden activation (tanh): the same kernel instantiations (the activation is a run-time
epilogue argument).

Each case also logs its launches (nf_debug_log_*) and checks that every kernel instantiation
+ variant a bench-identical call launches is among them.
"""
import numpy as np
import pytest
import torch

import synth
from oracle.batched import BatchedOracle
from parity import FP32_BAR, TF32_BAR, rel_err

pytestmark = pytest.mark.gpu

import paper_1902_06714_b200 as nf  # noqa: E402

MATH = {"fp32": nf.NF_MATH_FP32, "tf32": nf.NF_MATH_TF32}
# relu kink band (fraction of the layer's rms pre-activation): >= ~50x the measured error of
# the pre-activation sums in each mode (fp32: 3xTF32 / FFMA, TF32: RN-rounded operands)
MARGIN = {"fp32": 3e-5, "tf32": 1e-3}


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def launch_keys(lines):
    """kernel instantiation + variant of each logged launch (grid / smem dropped)"""
    keys = set()
    for l in lines:
        name, rest = l.split(" grid=", 1)
        note = rest.split(" smem=", 1)[1].split(" ", 1)
        keys.add((name, note[1] if len(note) > 1 else ""))
    return keys


def select_rows(o, p, cid, act, B, margin, pool_factor=16):
    """B kink-free rows of config cid's seeded inputs (pool of up to pool_factor * B rows)."""
    cfg = synth.CONFIGS[cid]
    N = min(cfg["N"], pool_factor * B)
    X, Y = synth.dataset(cid, N=N)
    if not any(a in act for a in ("relu", "step")):
        return X[:B], Y[:B]
    keep = np.zeros(N, bool)
    for r0 in range(0, N, B):
        _, Z = o.forward(p, X[r0:r0 + B])
        keep[r0:r0 + B] = o.kink_free_rows(Z, margin)
        if keep.sum() >= B:
            break
    idx = np.flatnonzero(keep)[:B]
    assert len(idx) == B, f"only {len(idx)} kink-free rows of {N}"
    return np.ascontiguousarray(X[idx]), np.ascontiguousarray(Y[idx])


def choose_eta(o, p, X, Y, rows=512):
    """eta such that the update is a sizeable fraction (~0.1-0.5) of the parameter scale in the
    layer where it is smallest, estimated from the tendencies of the first `rows` rows (the
    step is linear in eta; see module doc)."""
    G = o.grad(p, X[:rows], Y[:rows])
    r = []
    for (W, b), (gW, gb) in zip(o.layers(p.astype(np.float64)), o.layers(G)):
        r.append(np.abs(W).max() / max(np.abs(gW).max(), 1e-30))
        r.append(np.abs(b).max() / max(np.abs(gb).max(), 1e-30))
    return float(0.5 * min(rows, X.shape[0]) * min(r))


def update_err(got, ref, p0, nround, tau):
    """rel_err of the update (got - p0) vs (ref - p0) after removing nround half-ulps of the
    fp32 result from each element's difference."""
    got, ref, p0 = (np.asarray(a, np.float64) for a in (got, ref, p0))
    ulp = np.spacing(np.maximum(np.abs(ref), np.abs(got)).astype(np.float32)).astype(np.float64)
    d = np.maximum(np.abs(got - ref) - 0.5 * nround * ulp, 0.0)
    u = ref - p0
    scale = np.maximum(np.abs(u), tau * np.abs(u).max())
    scale = np.where(scale == 0, 1.0, scale)
    return float(np.max(d / scale))


CASES = [
    # (name, config id, activation override, dims override, math, batch)
    ("c3-fp32", 3, None, None, "fp32", 4096),
    ("c3-tf32", 3, None, None, "tf32", 4096),
    ("c4-fp32", 4, None, None, "fp32", 2048),
    ("c4-tf32", 4, None, None, "tf32", 2048),
    ("c5-fp32", 5, None, None, "fp32", 16384),
    ("c5w-tanh-tf32", 5, "tanh,sigmoid", None, "tf32", 16384),
]


@pytest.mark.parametrize("name,cid,act,dims,math,B", CASES, ids=[c[0] for c in CASES])
def test_full_size_step(name, cid, act, dims, math, B):
    cfg = synth.CONFIGS[cid]
    dims = dims or cfg["dims"]
    act = act or cfg["act"]
    p = synth.init_params(cid, dims)
    o = BatchedOracle(dims, act)
    X, Y = select_rows(o, p, cid, act, B, MARGIN[math])
    eta = choose_eta(o, p, X, Y)
    ref, ref_loss, _ = o.train_batch(p, X, Y, eta)

    net = nf.Net(dims, act)
    net.set_math(MATH[math])
    net.set_params(dev(p))
    loss = torch.zeros(1, device="cuda")
    nf.nf_debug_log_enable(True)
    net.train_steps(dev(X), dev(Y), B, [0], eta, step_loss=loss)
    torch.cuda.synchronize()
    tested = launch_keys(nf.nf_debug_log_read())
    got = net.get_params()

    tau, bar = (0.1, FP32_BAR) if math == "fp32" else (1.0, TF32_BAR)
    nW, nb = 8, B // 32 + 8   # in-place fp32 adds per element: split-K terms / bias strips
    errs = []
    for l, ((Wg, bg), (Wr, br), (W0, b0)) in enumerate(zip(o.layers(got), o.layers(ref), o.layers(p)), 1):
        eW, eb = update_err(Wg, Wr, W0, nW, tau), update_err(bg, br, b0, nb, tau)
        errs.append((l, eW, eb, update_err(Wg, Wr, W0, nW, 0.1), update_err(bg, br, b0, nb, 0.1)))
    print(f"{name}: eta {eta:.3g}; per layer (W, b) update err at tau={tau}, and at tau=0.1: " +
          "; ".join(f"L{l} {a:.2e} {b:.2e} ({c:.2e} {d:.2e})" for l, a, b, c, d in errs))
    for l, eW, eb, _, _ in errs:
        assert eW <= bar, (name, l, "W", eW)
        assert eb <= bar, (name, l, "b", eb)
    assert rel_err(loss.cpu().numpy(), [ref_loss]) <= (FP32_BAR if math == "fp32" else TF32_BAR)

    # coverage: a bench-identical call (config's dataset shape, bench's starts) launches
    # nothing this test did not
    Xb, Yb = synth.dataset(cid, N=min(cfg["N"], 2 * B + 64))
    starts = synth.batch_starts(cid, steps=2, N=len(Xb), batch=B)
    bench_net = nf.Net(dims, act)
    bench_net.set_math(MATH[math])
    bench_net.set_params(dev(p))
    nf.nf_debug_log_enable(True)
    bench_net.train_steps(dev(Xb), dev(Yb), B, starts, cfg["eta"], step_loss=torch.zeros(2, device="cuda"))
    torch.cuda.synchronize()
    bench = launch_keys(nf.nf_debug_log_read())
    nf.nf_debug_log_enable(False)
    missing = bench - tested
    assert not missing, f"bench launches not covered by {name}: {missing}"
    print(f"{name}: {len(tested)} kernel instantiations / variants covered: " +
          " | ".join(sorted(f"{k[0].replace('(anonymous namespace)::', '').split('(')[0]} [{k[1]}]" for k in tested)))
