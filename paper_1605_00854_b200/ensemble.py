"""Multi-GPU ensemble plumbing: trajectories are independent, so
global trajectory ids are split into contiguous per-rank ranges and the only
collective is ONE all-reduce (sum) of the pooled counts at the end. Because
every draw is keyed by (seed, global trajectory id, step), the totals are
identical for any rank count."""
from __future__ import annotations

import numpy as np

COUNT_FIELDS = 8


def shard_range(n_total: int, world: int, rank: int):
    """Contiguous [begin, begin+count) of global trajectory ids for `rank`."""
    base, extra = divmod(n_total, world)
    begin = rank * base + min(rank, extra)
    return begin, base + (1 if rank < extra else 0)


def pooled(counts) -> np.ndarray:
    """Per-trajectory count records (n, 8) -> pooled totals (8,) int64."""
    c = np.asarray(counts, dtype=np.uint64).reshape(-1, COUNT_FIELDS)
    return c.sum(axis=0, dtype=np.uint64).astype(np.int64)


def allreduce_totals(totals, device=None):
    """The single collective of the path: sum the pooled totals over ranks
    (NCCL on GPUs, gloo on CPU). No-op without an initialised process group."""
    import torch
    import torch.distributed as dist

    t = torch.as_tensor(np.asarray(totals, dtype=np.int64), device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().numpy()


def run_sharded(simulate, n_total: int, world: int, rank: int, device=None):
    """simulate(traj_begin, n_traj) -> per-trajectory counts (n_traj, 8).
    Returns the job-wide pooled totals (identical on every rank)."""
    begin, count = shard_range(n_total, world, rank)
    local = pooled(simulate(begin, count)) if count else np.zeros(COUNT_FIELDS, np.int64)
    return allreduce_totals(local, device)
