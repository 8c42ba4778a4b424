"""Multi-GPU plumbing for sweeps (one process per GPU, torch.distributed).

Replications are independent (experiment.hpp:5-8), so a sweep shards by
replication: rank r simulates replications [lo, hi) of every point into its
own block [6][points][hi - lo] (the C ABI's BB_REP_* fields,
bb_points_shard_local_device).  The sweep's ONE collective is an all-gather
of those blocks in rank order (each rank moves only its own slice, instead of
all-reducing a zero-padded copy of the whole array), and the per-point
mean/std (run_point, experiment.hpp:266-281) then runs over the gathered
blocks in replication order (bb_points_reduce_gathered_device) --
bit-identical to a single-process run.

``combine`` (the zero-padded full array + one all-reduce sum, x + 0 == x) is
kept for callers of bb_points_shard_device's full-array layout.
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


def block_index(field: int, point: int, rep: int, n_points: int, reps_total: int, world: int) -> int:
    """Flat index of (field, point, replication) in the gathered shard blocks
    (shard c holds [R c / W, R (c+1) / W) as [field][point][its replications])."""
    c = next(c for c in range(world) if reps_total * (c + 1) // world > rep)
    lo, hi = reps_total * c // world, reps_total * (c + 1) // world
    return REP_FIELDS * n_points * lo + (field * n_points + point) * (hi - lo) + (rep - lo)


def gather(block, out, group=None):
    """The sweep's single collective: every rank's block concatenated in rank
    order into `out` (world x block elements; `out` may be `block` at N=1)."""
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        if out.data_ptr() != block.data_ptr():
            out.copy_(block)
        return out
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, block, group=group)
    else:  # gloo: list form
        parts = list(out.chunk(dist.get_world_size(group)))
        dist.all_gather(parts, block, group=group)
    return out


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
