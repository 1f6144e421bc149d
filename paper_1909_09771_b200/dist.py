"""Multi-GPU batch sharding (one process per GPU, torch.distributed).

A single NTD-PCG system never spans GPUs: its sweeps are sequential in z and
y (ntd_solve.py:198-253).  A batch of independent systems (BASELINE config 4)
is sharded: rank r of W owns systems [B*r/W, B*(r+1)/W), builds them from
their seeds, solves them with no data-path communication, and the ranks
exchange only per-system statistics at the end (one all_gather) plus the
max-reduced timings.  Works with the NCCL backend on GPUs and gloo on CPU
(tests/test_dist_gloo.py).
"""

import torch
import torch.distributed as dist

STAT_FIELDS = ("system", "iterations", "converged", "final_relres")


def shard(total, world, rank):
    """Contiguous, balanced system range of `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return list(range(total * rank // world, total * (rank + 1) // world))


def gather_stats(rows, total, device=None):
    """All-gather per-system stat rows [(system, iters, converged, relres), ...]
    from every rank; returns a (total, 4) float64 tensor ordered by system."""
    device = device or torch.device("cpu")
    t = torch.tensor(rows, dtype=torch.float64, device=device).reshape(-1, len(STAT_FIELDS))
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        out = t
    else:
        world = dist.get_world_size()
        sizes = [len(shard(total, world, r)) for r in range(world)]
        pad = torch.zeros((max(sizes), len(STAT_FIELDS)), dtype=torch.float64, device=device)
        pad[: t.shape[0]] = t
        parts = [torch.zeros_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad)
        out = torch.cat([p[:sz] for p, sz in zip(parts, sizes)])
    order = torch.argsort(out[:, 0])
    return out[order]


def reduce_max(values, device=None):
    """Element-wise max over ranks (timings: the job time is the slowest rank)."""
    device = device or torch.device("cpu")
    t = torch.tensor(values, dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def reduce_sum(values, device=None):
    device = device or torch.device("cpu")
    t = torch.tensor(values, dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.tolist()
