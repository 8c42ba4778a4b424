"""The trace pipeline's CUDA graph: the sync-free pipeline is captured on the
second identical call (same sizes, same device pointers) and replayed from
the third.  A replay must give exactly the direct pipeline's results on new
data in the same buffers, new bin edges, and input errors.  Results are
checked against the oracle (the checker) like tests/test_gpu_trace.py."""
import math

import numpy as np
import pytest
import torch

import oracle_py as O
import paper_2412_04504_b200 as bb
from test_gpu_trace import check_metrics, sim_config

pytestmark = pytest.mark.gpu

N = 200_000


def _case(seed, k=8, B=16, load=0.95, edges=None, error="symmetric"):
    cfg = dict(arrival_rate=load * bb.throughput(B, k, 1.0, 20.0), n_requests=N, batch_size=B,
               edges=edges or bb.uniform_boundaries(k, 1.0, 20.0).edges, lo=1.0, hi=20.0,
               seed=seed, error=error, p_error=0.1)
    m, d = O.run(O.oracle(), cfg)
    u = O.stream_uniform01(O.oracle(), seed, 2, N) if error == "symmetric" else None
    return cfg, m, d, u


class Buffers:
    """Device-resident request arrays reused across calls (stable pointers)."""

    def __init__(self, tag):
        # distinct offsets per test: a fresh graph key even if the caching
        # allocator hands out the same blocks again
        off = 2 * tag
        self.a = torch.empty(N + off, dtype=torch.float64, device="cuda")[off:]
        self.s = torch.empty(N + off, dtype=torch.float64, device="cuda")[off:]
        self.u = torch.empty(N + off, dtype=torch.float64, device="cuda")[off:]
        self.stream = torch.cuda.Stream()

    def run(self, cfg, d, u):
        self.a.copy_(torch.from_numpy(d["req_arrival"]))
        self.s.copy_(torch.from_numpy(d["req_service"]))
        if u is not None:
            self.u.copy_(torch.from_numpy(u))
        torch.cuda.synchronize()
        return bb.run_trace_device(sim_config(cfg), self.a.data_ptr(), self.s.data_ptr(),
                                   self.u.data_ptr() if u is not None else 0,
                                   stream=self.stream.cuda_stream)


def _check(m, ref, d):
    lat = d["req_completion"] - d["req_arrival"]
    check_metrics(m, ref, N, np.nansum(np.abs(lat)), d["bat_service"].sum())


def test_replays_match_direct_runs_on_new_data():
    buf = Buffers(1)
    bb.trace_graph_stats(reset=True)
    cases = [_case(seed) for seed in (11, 12, 13, 14, 15)]
    for cfg, m, d, u in cases:
        _check(buf.run(cfg, d, u), m, d)
    captures, replays = bb.trace_graph_stats()
    assert captures == 1 and replays == 3  # direct, capture, 3 replays


def test_replay_uses_new_bin_edges_and_loads():
    """Edges are not part of the graph key (they are copied into graph-owned
    memory before each launch): a replay with other edges and another load
    must follow them."""
    buf = Buffers(2)
    bb.trace_graph_stats(reset=True)
    base = bb.uniform_boundaries(8, 1.0, 20.0).edges
    warped = [1.0] + [1.0 + 19.0 * (i / 8) ** 1.7 for i in range(1, 8)] + [20.0]
    seq = [_case(21, edges=base), _case(22, edges=base), _case(23, edges=warped, load=0.6),
           _case(24, edges=warped, load=1.2), _case(25, edges=base, load=0.99)]
    for cfg, m, d, u in seq:
        _check(buf.run(cfg, d, u), m, d)
    assert bb.trace_graph_stats() == (1, 3)


def test_replay_reports_input_errors_then_recovers():
    buf = Buffers(3)
    bb.trace_graph_stats(reset=True)
    cfg, m, d, u = _case(31)
    for _ in range(3):
        _check(buf.run(cfg, d, u), m, d)
    bad = dict(d)
    bad["req_arrival"] = d["req_arrival"].copy()
    bad["req_arrival"][N // 2] = 0.0  # non-monotone arrivals
    with pytest.raises(bb.InvalidArgument):
        buf.run(cfg, bad, u)
    bad["req_arrival"] = d["req_arrival"]
    bad["req_service"] = d["req_service"].copy()
    bad["req_service"][77] = 1e9  # outside the bins' support
    with pytest.raises(bb.DomainError):
        buf.run(cfg, bad, u)
    _check(buf.run(cfg, d, u), m, d)
    captures, replays = bb.trace_graph_stats()
    assert captures == 1 and replays == 4


def test_perfect_predictions_and_overload_replays():
    buf = Buffers(4)
    bb.trace_graph_stats(reset=True)
    for seed in (41, 42, 43):
        cfg, m, d, u = _case(seed, error="perfect", load=math.inf)
        _check(buf.run(cfg, d, u), m, d)
    assert bb.trace_graph_stats() == (1, 1)
