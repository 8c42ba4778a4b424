"""Multi-process sweep on the GPU: two ranks (gloo, sharing the one GPU of
the test box) simulate disjoint replication shards into their slices of the
per-replication array, ONE all-reduce assembles it, and the per-point
results are bit-identical to a single process running all replications."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

R = 64  # replications per rank


def points():
    import paper_2412_04504_b200 as bb
    return [bb.RunTemplate(arrival_rate=lam, n_requests=4000, batch_size=8, bins=bb.BinRule(k=k),
                           service=bb.ServiceSpec("uniform", 1.0, 20.0))
            for k in (1, 4) for lam in (0.3, 0.6)]


def _worker(rank, world, port, out):
    import torch.distributed as dist

    import paper_2412_04504_b200 as bb
    from paper_2412_04504_b200 import dist as bbdist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    pts = points()
    rtot = R * world
    rep = torch.zeros(6 * len(pts) * rtot, dtype=torch.float64, device="cuda")
    lo, hi = bbdist.weak_shard(R, rank)
    bb.points_shard_device(pts, rtot, 1234, lo, hi, rep.data_ptr())
    torch.cuda.synchronize()
    bbdist.combine(rep)
    torch.cuda.synchronize()
    res = bb.points_reduce_device(pts, rtot, rep.data_ptr())
    out[rank] = [(p.throughput_mean, p.throughput_std, p.latency_mean, p.latency_std) for p in res]
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sweep_equals_single_process():
    import paper_2412_04504_b200 as bb
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    single = bb.run_points(points(), 2 * R, 1234)
    want = [(p.throughput_mean, p.throughput_std, p.latency_mean, p.latency_std) for p in single]
    assert out[0] == want and out[1] == want
