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


def run_sharded_nodes(simulate, n_total: int, n_kept: int, world: int, rank: int, device=None):
    """simulate(traj_begin, n_traj) -> (counts (n_traj, 8), one-counts (n_traj, n_kept)).
    The job-wide pooled totals (8,) and pooled per-node one-counts (n_kept,),
    combined in ONE all-reduce of the concatenated vector (the C-ABI device
    group, csrc/group.cpp, does the same with one ncclAllReduce)."""
    begin, count = shard_range(n_total, world, rank)
    vec = np.zeros(COUNT_FIELDS + n_kept, np.int64)
    if count:
        cnt, nc = simulate(begin, count)
        vec[:COUNT_FIELDS] = pooled(cnt)
        vec[COUNT_FIELDS:] = np.asarray(nc, np.uint64).reshape(-1, n_kept).sum(
            axis=0, dtype=np.uint64).astype(np.int64)
    out = allreduce_totals(vec, device)
    return out[:COUNT_FIELDS], out[COUNT_FIELDS:]


# ----------------------------------------------------------------------------
# Pooled steady-state estimate across ranks ("the estimator does
# one all-reduce per round"). The C++ estimator (pbn_estimate_with_backend)
# runs identically on every rank; its backend steps this rank's shard and
# all-reduces the pooled counters, so every rank takes the same decisions.

class ShardedBackend:
    """stepper.run(step_begin, n, kappa, thin_mode, series_bit0|None, init) -> local
    totals (8,); stepper.stats(kappa, length) -> local series counters (13,)."""

    def __init__(self, stepper, device=None):
        self.stepper, self.device = stepper, device

    def run(self, s0, n, kappa, mode, bit0, init):
        return allreduce_totals(self.stepper.run(s0, n, kappa, mode, bit0, init), self.device)

    def stats(self, kappa, length):
        return allreduce_totals(np.asarray(self.stepper.stats(kappa, length), np.int64),
                                self.device)


def estimate_sharded(req, stepper, n_total: int, series_capacity: int, device=None):
    """Pooled estimate over n_total trajectories split across ranks."""
    from . import estimate_with_backend

    be = ShardedBackend(stepper, device)
    req.n_traj = n_total
    return estimate_with_backend(req, n_total, be.run, be.stats, series_capacity)


class DeviceShard:
    """One rank's trajectory shard on its GPU (torch tensors in HBM)."""

    def __init__(self, engine, pred, seed, traj_begin, n_traj, stream, series_capacity):
        import torch

        self.eng, self.pred, self.seed = engine, pred, seed
        self.tb, self.n, self.stream = traj_begin, n_traj, stream
        dev = torch.device("cuda", engine.device)
        self.states = torch.zeros((n_traj, engine.words), dtype=torch.int64, device=dev)
        self.counts = torch.zeros((n_traj, COUNT_FIELDS), dtype=torch.int64, device=dev)
        self.tprev = torch.zeros(n_traj, dtype=torch.uint8, device=dev)
        self.stride = (series_capacity + 31) // 32
        self.series = torch.zeros((n_traj, self.stride), dtype=torch.int32, device=dev)
        self.cs = torch.cuda.current_stream(dev)
        self.steps = 0

    def run(self, s0, n, kappa, mode, bit0, init):
        done = 0
        tot = np.zeros(COUNT_FIELDS, np.int64)
        while done < n:
            m = min(n - done, 1 << 31)
            self.eng.simulate_device(
                self.seed, self.n, m, self.states.data_ptr(), self.counts.data_ptr(),
                traj_begin=self.tb, step_begin=s0 + done, pred=self.pred, stream=self.stream,
                cuda_stream=self.cs.cuda_stream, kappa=kappa, thin_mode=mode if done == 0 else 1,
                d_tprev=self.tprev.data_ptr(),
                d_series=self.series.data_ptr() if bit0 is not None else None,
                series_stride=self.stride, series_bit0=(bit0 or 0) + done,
                series_init=init and done == 0)
            tot += self.counts.sum(dim=0).cpu().numpy()
            done += m
        self.steps += n
        return tot

    def stats(self, kappa, length):
        from . import series_stats_device

        self.cs.synchronize()
        return series_stats_device(self.eng.device, self.series.data_ptr(), self.n, self.stride,
                                   length, kappa).astype(np.int64)
