"""Multi-rank batch sharding and statistics gather (paper_1909_09771_b200.dist)
with world_size 2 over gloo on CPU -- the host-side logic of the multi-GPU
batch path (the GPU runs use NCCL with the same calls)."""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1909_09771_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = pdist.shard(total, world, rank)
    rows = [[s, 20 + s % 5, 1, 1e-9 * (s + 1)] for s in mine]
    stats = pdist.gather_stats(rows, total)
    tmax = pdist.reduce_max([float(rank + 1), 2.0 * rank])
    tsum = pdist.reduce_sum([float(len(mine))])
    if rank == 0:
        out.put((stats.tolist(), tmax, tsum))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_covers_batch_disjointly():
    for total in (1, 7, 64):
        for world in (1, 2, 4, 8):
            got = sorted(s for r in range(world) for s in pdist.shard(total, world, r))
            assert got == list(range(total))


def test_gloo_world2_gather_and_reduce():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    total = 7
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    stats, tmax, tsum = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert [int(r[0]) for r in stats] == list(range(total))
    assert [int(r[1]) for r in stats] == [20 + s % 5 for s in range(total)]
    assert tmax == [2.0, 2.0]
    assert tsum == [float(total)]


def test_single_process_fallbacks():
    rows = [[1, 5, 1, 0.1], [0, 4, 1, 0.2]]
    st = pdist.gather_stats(rows, 2)
    assert st[:, 0].tolist() == [0.0, 1.0]
    assert pdist.reduce_max([1.0, 3.0]) == [1.0, 3.0]
