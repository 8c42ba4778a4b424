"""Multi-GPU plumbing for sweeps (one process per GPU, torch.distributed).

Replications are independent (experiment.hpp:5-8), so a sweep shards by
replication: rank r owns replications [lo, hi) of every point and writes
them into its slice of a zero-initialised [6][points x R_total] float64
array (the C ABI's layout, BB_REP_*).  ONE all-reduce (sum) assembles the
full array -- x + 0 == x exactly, so the combined array is bit-identical to a
single-process run -- and the per-point mean/std (run_point,
experiment.hpp:266-281) is then computed in replication order.
"""
from __future__ import annotations

REP_FIELDS = 6


def weak_shard(reps_per_rank: int, rank: int):
    """Weak scaling: every rank adds reps_per_rank replications."""
    return rank * reps_per_rank, (rank + 1) * reps_per_rank


def strong_shard(reps_total: int, rank: int, world: int):
    """Strong scaling: a fixed replication count split contiguously."""
    return reps_total * rank // world, reps_total * (rank + 1) // world


def rep_index(field: int, point: int, rep: int, n_points: int, reps_total: int) -> int:
    """Flat index of (field, point, replication) in the per-replication array."""
    return field * n_points * reps_total + point * reps_total + rep


def combine(rep_tensor, group=None):
    """The sweep's single collective: sum the disjoint per-rank slices."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(rep_tensor, op=dist.ReduceOp.SUM, group=group)
    return rep_tensor


def mean_std(xs):
    """experiment.hpp:188-200 (sequential sum, sample std) -- host check helper."""
    n = float(len(xs))
    s = 0.0
    for x in xs:
        s += x
    mean = s / n
    if len(xs) < 2:
        return mean, 0.0
    ss = 0.0
    for x in xs:
        ss += (x - mean) * (x - mean)
    return mean, (ss / (n - 1.0)) ** 0.5
