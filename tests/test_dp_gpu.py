"""nf_update and the data-parallel driver on the GPU (-m gpu): one rank over NCCL (the pool
has one GPU per call; the two-rank co_sum logic is covered with gloo in test_dist_cpu.py)."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import synth
from parity import FP32_BAR, FP64_BAR, rel_err

pytestmark = pytest.mark.gpu

import paper_1902_06714_b200 as nf  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def params_of(net):
    out = torch.empty(net.n_params, dtype=torch.float32, device="cuda")
    net.get_params(out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("math", [nf.NF_MATH_FP32, nf.NF_MATH_FP64])
def test_update_applies_eta_over_n(math):
    """nf_update: params -= (eta / n) grad, device and host gradients."""
    dims = [37, 45, 13]
    p = synth.random_params(3, dims, 0.5).astype(np.float32)
    g = synth.random_params(4, dims, 2.0).astype(np.float32)
    net = nf.Net(dims, "tanh")
    net.set_params(dev(p))
    net.set_math(math)
    net.update(dev(g), 0.75, 30)
    ref = p.astype(np.float64) - (0.75 / 30) * g.astype(np.float64)
    assert rel_err(params_of(net), ref) <= (FP64_BAR if math == nf.NF_MATH_FP64 else 1e-6)
    net.update(g, 0.75, 30)                                  # host gradient
    ref = ref - (0.75 / 30) * g.astype(np.float64)
    assert rel_err(params_of(net), ref) <= (FP64_BAR if math == nf.NF_MATH_FP64 else 1e-6)
    with pytest.raises(nf.NFError):
        net.update(dev(g), 0.75, 0)
    with pytest.raises(nf.NFError):
        nf.nf_update(net.h, dev(g), net.n_params - 1, 0.75, 30)


def test_grad_then_update_equals_train_batch():
    """nf_grad + nf_update (the data-parallel step with one rank) == nf_train_batch."""
    dims = [784, 30, 10]
    p = synth.init_params(2)
    X, Y = synth.dataset(2, N=1000)
    a, b = nf.Net(dims, "sigmoid"), nf.Net(dims, "sigmoid")
    a.set_params(dev(p)); b.set_params(dev(p))
    a.train_batch(dev(X), dev(Y), 3.0)
    b.update(b.grad(dev(X), dev(Y)), 3.0, 1000)
    assert rel_err(params_of(b), params_of(a)) <= FP32_BAR


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_grad_layers_events_and_blocks():
    """nf_grad_layers writes the same tendencies as nf_grad and records one event per layer;
    a comm stream that waits on event l sees layer l's final block (the overlap contract)."""
    dims, act = [784, 1024, 1024, 10], "tanh"
    p = synth.init_params(3)
    X, Y = synth.dataset(3, N=4096)
    net = nf.Net(dims, act, stream=torch.cuda.current_stream())
    net.set_params(dev(p))
    ref = net.grad(dev(X), dev(Y)).clone()
    evs = [torch.cuda.Event() for _ in range(3)]
    for e in evs:
        e.record()
    g = torch.full_like(ref, float("nan"))
    comm = torch.cuda.Stream()
    copies = torch.empty_like(ref)
    net.grad_layers(dev(X), dev(Y), g, evs)
    with torch.cuda.stream(comm):
        for (off, cnt), e in zip(reversed(net.layer_slices()), reversed(evs)):
            comm.wait_event(e)
            copies[off:off + cnt].copy_(g[off:off + cnt])
    torch.cuda.synchronize()
    assert torch.isfinite(copies).all()
    assert rel_err(copies.cpu().numpy(), ref.cpu().numpy()) <= FP32_BAR
    with pytest.raises(nf.NFError):
        nf.nf_grad_layers(net.h, dev(X), dev(Y), 4096, g, evs[:2])


def test_data_parallel_one_rank_nccl():
    import torch.distributed as dist
    from paper_1902_06714_b200.dp import DataParallel
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        dims, act = [200, 136, 72, 5], "tanh"
        p = synth.random_params(51, dims, 0.1)
        X, Y = synth.random_batch(52, 600, dims[0], dims[-1], "uniform")
        starts = [0, 250, 100, 472]
        net = nf.Net(dims, act)
        net.set_params(dev(p))
        dp = DataParallel(net)
        dp.train_steps(dev(X), dev(Y), 128, starts, 0.5)
        ref, _ = oracle.Oracle(dims, act).train_steps(p, X, Y, 128, starts, 0.5)
        assert rel_err(params_of(net), ref) <= FP32_BAR
        net2 = nf.Net(dims, act)          # the same steps with the collectives not overlapped
        net2.set_params(dev(p))
        DataParallel(net2, overlap=False).train_steps(dev(X), dev(Y), 128, starts, 0.5)
        assert rel_err(params_of(net2), params_of(net)) <= 1e-6
    finally:
        dist.destroy_process_group()
