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
