"""The N > 1 host path of bench.py on CPU (gloo, world size 2, 127.0.0.1): max-over-ranks
timing and the whole-job aggregation (replicas only: the path does not shard across GPUs,
DESIGN.md section 8)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = [0.25, 0.40][rank]                      # per-rank device time of K steps
    t_max = bench.max_over_ranks(t, world)
    bench.barrier(world)
    q.put((rank, t_max, bench.job_throughput(world, 500, 1000, t_max)))
    dist.destroy_process_group()


def test_max_over_ranks_and_job_throughput_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, t_max, value in res:
        assert t_max == pytest.approx(0.40)            # the slowest rank decides
        assert value == pytest.approx(2 * 500 * 1000 / 0.40)


def test_single_rank_is_identity():
    import sys
    sys.path.insert(0, ROOT)
    import bench
    assert bench.max_over_ranks(0.3, 1) == 0.3
    assert bench.job_throughput(1, 10, 8, 0.5) == pytest.approx(160.0)


# ------------------------------------------------------------ data parallelism
class OracleNet:
    """CPU stand-in for nf.Net in the host-logic test of paper_1902_06714_b200.dp: the same
    method surface (grad / update / get_params / set_params), the arithmetic from the oracle,
    fp32 at the boundary like the C ABI."""

    def __init__(self, dims, act, params):
        import numpy as np
        import oracle
        self.o = oracle.Oracle(dims, act)
        self.p = np.asarray(params, dtype=np.float64)
        self.n_params = self.o.n_params

    def get_params(self, out):
        import torch
        out.copy_(torch.from_numpy(self.p.astype("float32")))

    def set_params(self, p):
        self.p = p.numpy().astype("float64")

    def grad(self, x, y, out):
        import torch
        out.copy_(torch.from_numpy(self.o.grad(self.p, x.numpy(), y.numpy()).astype("float32")))

    def grad_layers(self, x, y, out, events):
        assert len(events) == len(self.o.dims) - 1
        self.grad(x, y, out)

    def layer_slices(self):
        out, o = [], 0
        for l in range(1, len(self.o.dims)):
            c = self.o.dims[l] * self.o.dims[l - 1] + self.o.dims[l]
            out.append((o, c))
            o += c
        return out

    def update(self, g, eta, n):
        import numpy as np
        self.p = self.p - (float(np.float32(eta)) / n) * g.numpy().astype(np.float64)


def _dp_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import torch.distributed as dist
    import synth
    from paper_1902_06714_b200.dp import DataParallel
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dims, act = [13, 9, 7, 4], "tanh,sigmoid"
    p0 = synth.random_params(7, dims, 0.5).astype(np.float32).astype(np.float64)
    # only rank 0's initial parameters count: the co_broadcast must overwrite the others
    net = OracleNet(dims, act, p0 if rank == 0 else p0 + 1.0)
    dp = DataParallel(net, device="cpu")
    X, Y = synth.random_batch(8, 40, dims[0], dims[-1], "uniform")
    dp.train_steps(torch.from_numpy(X), torch.from_numpy(Y), 11, [0, 29, 5, 17], 0.8)
    dp.train_batch(torch.from_numpy(X[:1]), torch.from_numpy(Y[:1]), 0.8)   # 1 row < 2 ranks
    q.put((rank, net.p))
    dist.destroy_process_group()


def test_data_parallel_co_sum_equals_serial_gloo():
    """World size 2 (gloo): co_broadcast, per-rank tendencies of each rank's rows, co_sum as one
    all-reduce per layer block (layer L first: the bucketing the GPU path overlaps with the
    backward), identical update on every rank == the serial oracle on the whole batch
    (P:536-556)."""
    import sys
    sys.path.insert(0, ROOT)
    import numpy as np
    import oracle
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    dims, act = [13, 9, 7, 4], "tanh,sigmoid"
    p0 = synth.random_params(7, dims, 0.5).astype(np.float32).astype(np.float64)
    X, Y = synth.random_batch(8, 40, dims[0], dims[-1], "uniform")
    o = oracle.Oracle(dims, act)
    eta = float(np.float32(0.8))
    ref, _ = o.train_steps(p0, X, Y, 11, [0, 29, 5, 17], eta)
    ref, _ = o.train_batch(ref, X[:1], Y[:1], eta)
    assert np.array_equal(res[0], res[1])                       # every rank holds the same net
    scale = np.maximum(np.abs(ref), 0.1 * np.abs(ref).max())
    assert np.max(np.abs(res[0] - ref) / scale) <= 1e-6         # fp32 tendencies at the boundary


def test_shard_partitions_rows():
    import sys
    sys.path.insert(0, ROOT)
    from paper_1902_06714_b200.dp import shard
    for n in (1, 2, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            parts = [shard(n, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in parts]
            assert max(sizes) - min(sizes) <= 1
