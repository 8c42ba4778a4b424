"""Multi-GPU sweeps on the one GPU of the test box, bit-identical to a single
run of all replications:
* two processes (gloo) simulate disjoint replication shards into their own
  blocks, ONE all-gather assembles them, the gathered reduce runs in
  replication order (bench.py's protocol); the legacy full-array all-reduce;
* one process, several logical devices through the C ABI (bb_set_devices):
  one host thread per shard, results stored into devices[0]'s gather array."""
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
    lo, hi = bbdist.weak_shard(R, rank)
    # the gather protocol: own block, one all-gather, gathered reduce
    block = torch.empty(6 * len(pts) * R, dtype=torch.float64, device="cuda")
    bb.points_shard_local_device(pts, rtot, 1234, lo, hi, block.data_ptr())
    torch.cuda.synchronize()
    gathered = torch.empty(world * block.numel(), dtype=torch.float64, device="cuda")
    bbdist.gather(block, gathered)
    torch.cuda.synchronize()
    res = bb.points_reduce_gathered_device(pts, rtot, world, gathered.data_ptr())
    # the legacy full-array all-reduce
    rep = torch.zeros(6 * len(pts) * rtot, dtype=torch.float64, device="cuda")
    bb.points_shard_device(pts, rtot, 1234, lo, hi, rep.data_ptr())
    torch.cuda.synchronize()
    bbdist.combine(rep)
    torch.cuda.synchronize()
    res2 = bb.points_reduce_device(pts, rtot, rep.data_ptr())
    out[rank] = ([(p.throughput_mean, p.throughput_std, p.latency_mean, p.latency_std, p.latency_p50,
                   p.latency_p99) for p in res],
                 [(p.throughput_mean, p.throughput_std, p.latency_mean, p.latency_std, p.latency_p50,
                   p.latency_p99) for p in res2])
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
    want = [(p.throughput_mean, p.throughput_std, p.latency_mean, p.latency_std, p.latency_p50,
             p.latency_p99) for p in single]
    for rank in range(2):
        assert out[rank][0] == want  # gather protocol
        assert out[rank][1] == want  # all-reduce protocol


def _fields(res):
    return [(p.throughput_mean, p.throughput_std, p.latency_mean, p.latency_std, p.latency_p50,
             p.latency_p99, p.makespan_mean, p.busy_fraction_mean) for p in res]


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0]])
def test_c_abi_device_list_equals_one_device(devices):
    """bb_set_devices: one host thread per shard, results bit-identical to one
    device (shards on the one test GPU run on separate streams)."""
    import paper_2412_04504_b200 as bb
    pts = points()
    one = _fields(bb.run_points(pts, 97, 4321))
    try:
        bb.set_devices(devices)
        many = _fields(bb.run_points(pts, 97, 4321))
        spec = bb.ExperimentSpec(base=pts[0], axes=[bb.SweepAxis("k", [1, 2, 4])], replications=50, seed=9)
        exp_many = _fields(bb.run_experiment(spec))
    finally:
        bb.set_devices([])
    assert many == one
    assert exp_many == _fields(bb.run_experiment(spec))


def test_c_abi_device_list_errors():
    import paper_2412_04504_b200 as bb
    with pytest.raises(bb.InvalidArgument):
        bb.set_devices([0, 99])
    bad = bb.RunTemplate(arrival_rate=0.5, n_requests=1000, batch_size=8, bins=bb.BinRule(edges=[1.0, 5.0, 10.0]),
                         service=bb.ServiceSpec("uniform", 1.0, 20.0))
    try:
        bb.set_devices([0, 0])
        with pytest.raises(bb.DomainError):  # binning.hpp:135-140 from a shard thread
            bb.run_points([bad], 8, 1)
    finally:
        bb.set_devices([])


def test_stream_ordered_shard_reports_errors_at_reduce():
    """bb_points_shard_device no longer synchronises: a device-side error is
    raised by the reduce that follows on the same device."""
    import paper_2412_04504_b200 as bb
    bad = bb.RunTemplate(arrival_rate=0.5, n_requests=1000, batch_size=8, bins=bb.BinRule(edges=[1.0, 5.0, 10.0]),
                         service=bb.ServiceSpec("uniform", 1.0, 20.0))
    rep = torch.zeros(6 * 8, dtype=torch.float64, device="cuda")
    bb.points_shard_device([bad], 8, 1, 0, 8, rep.data_ptr())  # returns without raising
    with pytest.raises(bb.DomainError):
        bb.points_reduce_device([bad], 8, rep.data_ptr())
    good = points()
    rep = torch.zeros(6 * len(good) * 8, dtype=torch.float64, device="cuda")
    bb.points_shard_device(good, 8, 1, 0, 8, rep.data_ptr())
    bb.points_reduce_device(good, 8, rep.data_ptr())  # the pending flag was cleared
