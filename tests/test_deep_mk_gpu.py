"""The deep-net task megakernel (csrc/deep_mk.cu, opt-in NF_DEEP_MK=1, TF32 nets of narrow hidden
layers such as config 4) against the
fp64 oracle (-m gpu): several SGD steps in ONE launch of nf_train_steps, per-step costs and the
applied updates at the TF32 bar (5e-3 normwise, reading R14b), on nets with ragged input widths,
hidden widths 64..256, one activation per layer and narrow output layers; plus its launch
signature (one launch per call) from the launch log.  Smooth activations: no relu kink
decisions (R8, R20; config 4 itself is covered at full size by tests/test_fullsize_gpu.py)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from parity import TF32_BAR, rel_err

pytestmark = pytest.mark.gpu

import paper_1902_06714_b200 as nf  # noqa: E402

CASES = [
    ([256, 128, 192, 64, 10], "tanh,sigmoid", 512, 3),
    ([100, 256, 256, 256, 7], "tanh,gaussian,tanh,sigmoid", 384, 4),
    ([784, 256, 256, 10], "sigmoid", 1024, 2),
    ([64, 64, 16], "tanh,sigmoid", 1024, 5),
]


@pytest.mark.parametrize("dims,act,batch,steps", CASES)
def test_deep_megakernel_steps(dims, act, batch, steps, monkeypatch):
    monkeypatch.setenv("NF_DEEP_MK", "1")   # opt-in path (read per call)
    p = synth.random_params(601 + len(dims), dims, 0.08)
    X, Y = synth.random_batch(602, 3 * batch, dims[0], dims[-1], "uniform")
    starts = np.random.default_rng(603).integers(0, 2 * batch + 1, size=steps)
    net = nf.Net(dims, act)
    net.set_math(nf.NF_MATH_TF32)
    net.set_params(torch.from_numpy(p).cuda())
    loss = torch.zeros(steps, device="cuda")
    nf.nf_debug_log_enable(True)
    net.train_steps(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), batch, starts, 0.7, step_loss=loss)
    torch.cuda.synchronize()
    log = nf.nf_debug_log_read()
    nf.nf_debug_log_enable(False)
    # one megakernel launch for all steps (after the first TF32 rounding of the weights)
    assert sum("deep_mk_kernel" in l for l in log) == 1 and all("deep_mk_kernel" in l or "round_tf32" in l for l in log), log
    got = net.get_params().astype(np.float64)
    ref, ref_loss = oracle.Oracle(dims, act).train_steps(p, X, Y, batch, starts, 0.7)
    p64 = p.astype(np.float64)
    e_upd = rel_err(got - p64, ref - p64, tau=1.0)
    e_loss = rel_err(loss.cpu().numpy(), ref_loss, tau=1.0)
    print(f"{dims} {act}: update err {e_upd:.2e} (normwise), step-cost err {e_loss:.2e}")
    assert e_upd <= TF32_BAR
    assert e_loss <= TF32_BAR
