"""Data-parallel training over torch.distributed ranks: the paper's scheme.

  1. co_broadcast: rank 0's initial parameters are broadcast to every rank.
  2. Each rank computes the weight and bias tendencies of ITS piece of the batch (the batch
     "evenly distributed between the parallel processors"): ``nf_grad_layers``.
  3. co_sum: the tendencies are summed over all ranks, one all-reduce(sum) per
     layer block of the flat tendency vector (NCCL over NVLink on the GPU box; gloo in the CPU
     tests).  On the GPU the blocks are reduced on a communication stream as the backward
     pass finishes them -- layer L first -- so the collectives of layers L..l+1 overlap the
     backward of layers l..1 (the library records one CUDA event per finished layer).
  4. Every rank applies the same update to its own copy: ``nf_update`` with the
     whole batch's eta / B scale (reading R3), ordered after the last collective.

One process per GPU; every rank passes the same global batch (or the same dataset and
batch starts) and takes its contiguous share of the rows.  The arithmetic runs in the
library's CUDA kernels; this module only partitions rows, orders streams and calls the
collectives.  ``net`` is any object with the ``Net`` methods used here (grad_layers,
layer_slices, update, get_params, set_params, n_params); the multi-rank CPU tests drive it
with a test-side stand-in.
"""
import torch
import torch.distributed as dist


def shard(n: int, world: int, rank: int):
    """Rows [lo, hi) of an n-row batch owned by `rank`: contiguous, sizes differ by <= 1."""
    return rank * n // world, (rank + 1) * n // world


class DataParallel:
    def __init__(self, net, group=None, device="cuda", overlap: bool = True):
        self.net = net
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = device
        self.g = torch.empty(net.n_params, dtype=torch.float32, device=device)
        self.slices = net.layer_slices()
        self.cuda = str(device).startswith("cuda")
        self.overlap = overlap and self.cuda
        if self.cuda:
            self.comm = torch.cuda.Stream()
            self.events = [torch.cuda.Event() for _ in self.slices]
            for e in self.events:          # materialise the cudaEvent_t handles
                e.record()
        else:
            self.comm, self.events = None, [None] * len(self.slices)
        self.broadcast_params()

    def broadcast_params(self):
        """co_broadcast of rank 0's parameters."""
        p = torch.empty(self.net.n_params, dtype=torch.float32, device=self.device)
        self.net.get_params(p)
        dist.broadcast(p, src=dist.get_global_rank(self.group, 0) if self.group else 0, group=self.group)
        self.net.set_params(p)

    def _co_sum(self):
        """All-reduce(sum) of each layer's block, layer L first; on the GPU on the comm stream,
        each after its layer's event (overlapping the rest of the backward pass)."""
        if not self.overlap:
            for off, cnt in reversed(self.slices):
                dist.all_reduce(self.g[off:off + cnt], op=dist.ReduceOp.SUM, group=self.group)
            return
        main = torch.cuda.current_stream()
        with torch.cuda.stream(self.comm):
            for (off, cnt), ev in zip(reversed(self.slices), reversed(self.events)):
                self.comm.wait_event(ev)
                dist.all_reduce(self.g[off:off + cnt], op=dist.ReduceOp.SUM, group=self.group)
        main.wait_stream(self.comm)

    def train_batch(self, x, y, eta: float):
        """One synchronous SGD step on the global batch (x, y): local tendencies, co_sum,
        update with eta / len(x)."""
        n = x.shape[0]
        if n < 1:
            raise ValueError("train needs n >= 1 (S:181)")
        lo, hi = shard(n, self.world, self.rank)
        if hi > lo:
            self.net.grad_layers(x[lo:hi], y[lo:hi], self.g, self.events if self.overlap else [None] * len(self.slices))
        else:                               # more ranks than rows: this rank adds nothing
            self.g.zero_()
            if self.overlap:
                for e in self.events:
                    e.record()
        self._co_sum()
        self.net.update(self.g, eta, n)

    def train_steps(self, X, Y, batch: int, starts, eta: float):
        """The paper's minibatch loop: for each start s the global batch is
        rows [s, s + batch) of the (replicated) dataset."""
        for s in starts:
            s = int(s)
            self.train_batch(X[s:s + batch], Y[s:s + batch], eta)
