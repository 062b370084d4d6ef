"""Data-parallel training over torch.distributed ranks: the paper's scheme.

  1. co_broadcast: rank 0's initial parameters are broadcast to every rank.
  2. Each rank computes the weight and bias tendencies of ITS piece of the batch (the batch
     "evenly distributed between the parallel processors"): ``nf_grad``.
  3. co_sum: the tendencies are summed over all ranks: one all-reduce(sum) of
     the flat tendency vector (NCCL over NVLink on the GPU box; gloo in the CPU tests).
  4. Every rank applies the same update to its own copy: ``nf_update`` with the
     whole batch's eta / B scale (reading R3).

One process per GPU; every rank passes the same global batch (or the same dataset and
batch starts) and takes its contiguous share of the rows.  The arithmetic runs in the
library's CUDA kernels; this module only partitions rows and calls the collective.
``net`` is any object with the ``Net`` methods used here (grad, update, get_params,
set_params, n_params); the multi-rank CPU tests drive it with a test-side stand-in.
"""
import torch
import torch.distributed as dist


def shard(n: int, world: int, rank: int):
    """Rows [lo, hi) of an n-row batch owned by `rank`: contiguous, sizes differ by <= 1."""
    return rank * n // world, (rank + 1) * n // world


class DataParallel:
    def __init__(self, net, group=None, device="cuda"):
        self.net = net
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = device
        self.g = torch.empty(net.n_params, dtype=torch.float32, device=device)
        self.broadcast_params()

    def broadcast_params(self):
        """co_broadcast of rank 0's parameters."""
        p = torch.empty(self.net.n_params, dtype=torch.float32, device=self.device)
        self.net.get_params(p)
        dist.broadcast(p, src=dist.get_global_rank(self.group, 0) if self.group else 0, group=self.group)
        self.net.set_params(p)

    def train_batch(self, x, y, eta: float):
        """One synchronous SGD step on the global batch (x, y): local tendencies, co_sum,
        update with eta / len(x)."""
        n = x.shape[0]
        if n < 1:
            raise ValueError("train needs n >= 1 (S:181)")
        lo, hi = shard(n, self.world, self.rank)
        if hi > lo:
            self.net.grad(x[lo:hi], y[lo:hi], self.g)
        else:                               # more ranks than rows: this rank adds nothing
            self.g.zero_()
        dist.all_reduce(self.g, op=dist.ReduceOp.SUM, group=self.group)
        self.net.update(self.g, eta, n)

    def train_steps(self, X, Y, batch: int, starts, eta: float):
        """The paper's minibatch loop: for each start s the global batch is
        rows [s, s + batch) of the (replicated) dataset."""
        for s in starts:
            s = int(s)
            self.train_batch(X[s:s + batch], Y[s:s + batch], eta)
