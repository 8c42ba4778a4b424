"""World-size-2 gloo runs of the sweep's multi-process protocol on CPU: shard
replications, fill each rank's block (or its slice of the full array), one
collective (all-gather of the blocks; the legacy all-reduce), per-point
mean/std in replication order -- identical to the single-process array and
statistics."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_04504_b200 import dist as bbdist

P, R = 5, 7  # points, replications per rank


def fake_metric(field, point, rep):
    # any deterministic per-(point, replication) value stands in for the kernel
    return 1.0 + 0.1 * field + point * 0.37 + (rep * 2654435761 % 1000) / 997.0


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rtot = R * world
    rep = torch.zeros(bbdist.REP_FIELDS * P * rtot, dtype=torch.float64)
    lo, hi = bbdist.weak_shard(R, rank)
    for f in range(bbdist.REP_FIELDS):
        for p in range(P):
            for r in range(lo, hi):
                rep[bbdist.rep_index(f, p, r, P, rtot)] = fake_metric(f, p, r)
    bbdist.combine(rep)
    stats = []
    for p in range(P):
        xs = [rep[bbdist.rep_index(0, p, r, P, rtot)].item() for r in range(rtot)]
        stats.append(bbdist.mean_std(xs))
    out[rank] = (rep.numpy().tobytes(), stats)
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_two_rank_shard_allreduce_matches_single_process():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, free_port(), out), nprocs=world, join=True)
    rtot = R * world
    full = torch.zeros(bbdist.REP_FIELDS * P * rtot, dtype=torch.float64)
    for f in range(bbdist.REP_FIELDS):
        for p in range(P):
            for r in range(rtot):
                full[bbdist.rep_index(f, p, r, P, rtot)] = fake_metric(f, p, r)
    for rank in range(world):
        blob, stats = out[rank]
        assert blob == full.numpy().tobytes()  # bit-identical assembly
        for p in range(P):
            xs = [full[bbdist.rep_index(0, p, r, P, rtot)].item() for r in range(rtot)]
            assert stats[p] == bbdist.mean_std(xs)


def test_shard_ranges_cover_exactly():
    for world in (1, 2, 3, 8):
        total = 10_000
        seen = []
        for r in range(world):
            lo, hi = bbdist.strong_shard(total, r, world)
            seen.extend(range(lo, hi))
        assert seen == list(range(total))
        assert bbdist.weak_shard(100, 3) == (300, 400)


def _gather_worker(rank, world, port, reps_total, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = bbdist.strong_shard(reps_total, rank, world)
    # every rank's block must have the same size for the all-gather: weak shards
    assert hi - lo == reps_total // world
    block = torch.empty(bbdist.REP_FIELDS * P * (hi - lo), dtype=torch.float64)
    for f in range(bbdist.REP_FIELDS):
        for p in range(P):
            for r in range(lo, hi):
                block[(f * P + p) * (hi - lo) + (r - lo)] = fake_metric(f, p, r)
    gathered = torch.empty(world * block.numel(), dtype=torch.float64)
    bbdist.gather(block, gathered)
    stats = []
    for p in range(P):
        xs = [gathered[bbdist.block_index(0, p, r, P, reps_total, world)].item()
              for r in range(reps_total)]
        stats.append(bbdist.mean_std(xs))
    out[rank] = (gathered.numpy().tobytes(), stats)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gather_of_blocks_matches_single_process():
    """bench.py's protocol: bb_points_shard_local_device blocks, one
    all-gather, the gathered reduce's replication order."""
    world, reps_total = 2, 2 * R
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gather_worker, args=(world, free_port(), reps_total, out), nprocs=world, join=True)
    for rank in range(world):
        blob, stats = out[rank]
        g = torch.frombuffer(bytearray(blob), dtype=torch.float64)
        for f in range(bbdist.REP_FIELDS):
            for p in range(P):
                for r in range(reps_total):
                    assert g[bbdist.block_index(f, p, r, P, reps_total, world)].item() == fake_metric(f, p, r)
        for p in range(P):
            assert stats[p] == bbdist.mean_std([fake_metric(0, p, r) for r in range(reps_total)])


def test_block_index_is_a_bijection():
    for world, total in ((1, 7), (2, 14), (3, 10), (8, 29)):
        idx = sorted(bbdist.block_index(f, p, r, P, total, world)
                     for f in range(bbdist.REP_FIELDS) for p in range(P) for r in range(total))
        assert idx == list(range(bbdist.REP_FIELDS * P * total))
