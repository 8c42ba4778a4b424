"""run_simulation / replay_trace with the reference's own random streams
(rng="reference"): the B200 engine reproduces the reference binary's
SimResult bit-for-bit (scalar sums within the reassociation bound)."""
import math

import numpy as np
import pytest

import oracle_py as O
import paper_2412_04504_b200 as bb
from _helpers import same_bits, sum_tol

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.have_reference(), reason="reference shim not built")]


CASES = [
    dict(arrival_rate=0.95 * 1.385550, n_requests=50000, batch_size=16, k=8, seed=1001,
         error=("symmetric", 0.1)),
    dict(arrival_rate=math.inf, n_requests=12800, batch_size=128, k=3, seed=77, flush=False),
    dict(arrival_rate=math.inf, n_requests=12807, batch_size=128, k=5, seed=78, flush=True,
         error=("symmetric", 0.25)),
    dict(arrival_rate=3.0, n_requests=2000, batch_size=8, k=3, seed=11,
         error=("confusion", [[0.7, 0.25, 0.05], [0.15, 0.7, 0.15], [0.02, 0.28, 0.7]])),
    dict(arrival_rate=7.0, n_requests=997, batch_size=13, k=3, seed=90210,
         error=("symmetric", 0.15)),
    # multi-server FIFO dispatch (simulator.hpp:256-277): acceptance criteria 3/9 shapes
    dict(arrival_rate=0.9 * 2 * 1.385550, n_requests=40000, batch_size=16, k=8, seed=2024,
         servers=2),
    dict(arrival_rate=0.8 * 64 * 0.6447481452557596, n_requests=30000, batch_size=4, k=4,
         seed=3, servers=64, error=("symmetric", 0.05)),
    dict(arrival_rate=math.inf, n_requests=12807, batch_size=32, k=5, seed=79, flush=True,
         servers=7),
    dict(arrival_rate=math.inf, n_requests=6400, batch_size=8, k=3, seed=80, flush=False,
         servers=3000),  # heap beyond shared memory
    # max_batch_wait (simulator.hpp:200-201,223-235): test_simulator.cpp:244-263 shape ...
    dict(arrival_rate=2.0, n_requests=400, batch_size=10, k=4, seed=70, servers=8, mbw=1.5),
    # ... and larger: timers and full batches mixed, flush / no flush, errors, 3 servers
    dict(arrival_rate=1.2, n_requests=60000, batch_size=16, k=8, seed=5, mbw=9.0,
         error=("symmetric", 0.1)),
    dict(arrival_rate=0.7, n_requests=30001, batch_size=32, k=4, seed=6, mbw=4.0, flush=False),
    dict(arrival_rate=2.5, n_requests=20000, batch_size=8, k=3, seed=7, mbw=0.75, servers=3),
    dict(arrival_rate=0.2, n_requests=5000, batch_size=4, k=1, seed=8, mbw=30.0),
    dict(arrival_rate=math.inf, n_requests=12807, batch_size=128, k=5, seed=81, flush=True,
         mbw=2.0),  # overload + flush: every bin drains at t = 0, the timers go stale
    # overload without flush: the partial batches form when their timers fire at W,
    # in arming order (first arrivals, then each bin's last round-robin formation)
    dict(arrival_rate=math.inf, n_requests=12807, batch_size=128, k=5, seed=82, flush=False,
         mbw=2.0),
    dict(arrival_rate=math.inf, n_requests=3003, batch_size=256, k=8, seed=83, flush=False,
         mbw=1e5, error=("symmetric", 0.2)),  # bins that never fill a batch; idle until W
    dict(arrival_rate=math.inf, n_requests=9001, batch_size=64, k=4, seed=84, flush=False,
         mbw=3.0, servers=3),
]


def configs(c):
    edges = bb.uniform_boundaries(c["k"], 1.0, 20.0).edges
    em, od = bb.Perfect(), {}
    if "error" in c:
        kind, p = c["error"]
        if kind == "symmetric":
            em, od = bb.Symmetric(p), dict(error="symmetric", p_error=p)
        else:
            em, od = bb.Confusion(p), dict(error="confusion", confusion=p)
    ours = bb.SimConfig(arrival_rate=c["arrival_rate"], n_requests=c["n_requests"],
                        batch_size=c["batch_size"], bins=bb.BinConfig(edges), error_model=em,
                        service=bb.Uniform(1.0, 20.0), seed=c["seed"],
                        flush_partial=c.get("flush", True), rng="reference",
                        n_servers=c.get("servers", 1), max_batch_wait=c.get("mbw"))
    ref = dict(arrival_rate=c["arrival_rate"], n_requests=c["n_requests"],
               batch_size=c["batch_size"], edges=edges, lo=1.0, hi=20.0, seed=c["seed"],
               flush_partial=c.get("flush", True), n_servers=c.get("servers", 1),
               max_batch_wait=c.get("mbw"), **od)
    return ours, ref


@pytest.mark.parametrize("i", range(len(CASES)))
def test_run_simulation_detailed_matches_reference_binary(i):
    ours, ref = configs(CASES[i])
    mr, dr = O.run(O.reference(), ref)
    res = bb.run_simulation_detailed(ours)
    r, b = res.requests, res.batches
    assert same_bits(r["arrival"], dr["req_arrival"])
    assert same_bits(r["service"], dr["req_service"])
    assert same_bits(r["true_bin"], dr["req_true_bin"])
    assert same_bits(r["predicted_bin"], dr["req_pred_bin"])
    assert same_bits(r["completion"], dr["req_completion"])
    assert same_bits(b["finish_time"], dr["bat_finish"])
    assert same_bits(b["start_time"], dr["bat_start"])
    assert same_bits(b["formed_time"], dr["bat_formed"])
    assert same_bits(b["members"], dr["members"])
    assert same_bits(b["size"], dr["bat_size"]) and same_bits(b["bin"], dr["bat_bin"])
    served = dr["req_batch"] != np.uint64(2**64 - 1)  # kNoBatch (simulator.hpp:35)
    assert np.array_equal(np.asarray(r["batch"])[served].astype(np.uint64), dr["req_batch"][served])
    if c_mbw := CASES[i].get("mbw"):  # the reference's own timer test (test_simulator.cpp:257-262)
        assert res.metrics.n_completed == ours.n_requests
        formed = np.asarray(b["formed_time"])[np.asarray(r["batch"], dtype=np.int64)]
        assert np.all(formed - np.asarray(r["arrival"]) <= c_mbw + 1e-9)
    m = res.metrics
    n = ours.n_requests
    for key in ("makespan", "throughput", "latency_p50", "latency_p99"):
        assert same_bits(getattr(m, key), mr[key]), key
    if ours.n_servers > 1:  # busy_time_ accumulates in dispatch order: exact
        assert same_bits(m.server_busy_fraction, mr["server_busy_fraction"])
    else:
        assert abs(m.server_busy_fraction - mr["server_busy_fraction"]) <= 1e-10
    lat = dr["req_completion"] - dr["req_arrival"]
    assert abs(m.latency_mean - mr["latency_mean"]) <= sum_tol(n, np.nansum(np.abs(lat))) / mr["n_completed"]
    # metrics-only entry agrees with the detailed one
    m2 = bb.run_simulation(ours)
    assert same_bits(m2.throughput, m.throughput) and same_bits(m2.latency_p99, m.latency_p99)


def test_replay_trace_resample_matches_reference():
    # acceptance.cpp criterion 10 setting (Pareto-like trace, B=32, overload, resample)
    trace = O.acceptance_trace()  # acceptance.cpp:366-375
    for k in (1, 4, 16, 32):
        edges = bb.empirical_boundaries(k, trace).edges
        seed = bb.replication_seed(1001, 3)
        ours = bb.SimConfig(arrival_rate=bb.kOverload, n_requests=12800, batch_size=32,
                            bins=bb.BinConfig(edges), seed=seed, flush_partial=False,
                            trace_mode="resample", rng="reference")
        mr, dr = O.run(O.reference(), dict(arrival_rate=math.inf, n_requests=12800, batch_size=32,
                                           edges=edges, seed=seed, flush_partial=False,
                                           service="trace_resample", table=trace))
        m = bb.replay_trace(ours, trace)
        assert same_bits(m.throughput, mr["throughput"])
        assert same_bits(m.latency_p50, mr["latency_p50"])


def test_run_experiment_reference_streams_bit_exact_throughput():
    # acceptance criterion 1 protocol (B=128, U[1,20], overload, no flush, 10 seeds)
    base = bb.RunTemplate(n_requests=12800, batch_size=128, flush_partial=False,
                          service=bb.ServiceSpec("uniform", 1.0, 20.0))
    spec = bb.ExperimentSpec(base=base, axes=[bb.SweepAxis("k", [1, 2, 3, 5])], replications=10,
                             seed=1001, rng="reference")
    pts = bb.run_experiment(spec)
    want = {1: 6.447, 2: 8.438, 3: 9.392, 5: 10.34}  # proj/test_output.txt:17
    for p in pts:
        assert f"{p.throughput_mean:.4g}" == f"{want[p.k]:.4g}"
        ref_thr = []
        for r in range(10):
            mr, _ = O.run(O.reference(), dict(arrival_rate=math.inf, n_requests=12800,
                                              batch_size=128,
                                              edges=bb.uniform_boundaries(p.k, 1.0, 20.0).edges,
                                              lo=1.0, hi=20.0, seed=bb.replication_seed(1001, r),
                                              flush_partial=False), detail=False)
            ref_thr.append(mr["throughput"])
        mean = 0.0
        for x in ref_thr:
            mean += x
        mean /= 10
        assert same_bits(p.throughput_mean, mean)


def test_acceptance_criterion3_multi_server_reference_streams():
    # acceptance.cpp:126-165: 64 servers, B=128, U[1,20], flush, lambda x k grid,
    # 10 seeds; published "lambda=10 k=1: measured 26.24 vs 26.2" (test_output.txt:19)
    base = bb.RunTemplate(n_requests=12800, batch_size=128, n_servers=64, flush_partial=True,
                          service=bb.ServiceSpec("uniform", 1.0, 20.0))
    spec = bb.ExperimentSpec(base=base, axes=[bb.SweepAxis("lambda", [5.0, 10.0]),
                                              bb.SweepAxis("k", [1, 2, 3])],
                             replications=10, seed=1001, rng="reference")
    pts = bb.run_experiment(spec)
    assert f"{pts[3].latency_mean:.4g}" == "26.24"
    for p in pts:
        pred = bb.expected_latency(128, p.k, 1.0, 20.0, p.arrival_rate)
        assert abs(p.latency_mean - pred) / pred < 0.05
        thr = []
        for r in range(10):
            mr, _ = O.run(O.reference(), dict(arrival_rate=p.arrival_rate, n_requests=12800,
                                              batch_size=128, n_servers=64,
                                              edges=bb.uniform_boundaries(p.k, 1.0, 20.0).edges,
                                              lo=1.0, hi=20.0, seed=bb.replication_seed(1001, r)),
                          detail=False)
            thr.append(mr["throughput"])
        mean = 0.0
        for x in thr:
            mean += x
        assert same_bits(p.throughput_mean, mean / 10)


def test_acceptance_criterion10_curve_exact():
    # acceptance.cpp:366-395 with the reference's streams: the published
    # curve 0.6538 0.807 1.009 1.338 1.751 2.355 (proj/test_output.txt:26)
    trace = O.acceptance_trace().tolist()
    base = bb.RunTemplate(n_requests=12800, batch_size=32, flush_partial=False,
                          service=bb.ServiceSpec("trace", trace_times=trace, trace_mode="resample"))
    spec = bb.ExperimentSpec(base=base, axes=[bb.SweepAxis("k", [1, 2, 4, 8, 16, 32])],
                             replications=10, seed=1001, rng="reference")
    got = [f"{p.throughput_mean:.4g}" for p in bb.run_experiment(spec)]
    assert got == ["0.6538", "0.807", "1.009", "1.338", "1.751", "2.355"]


def test_run_point_reference_streams_with_timers_bit_exact():
    # run_point (experiment.hpp:254-307) with max_batch_wait over the
    # reference's own streams: per-replication metrics equal the binary's
    t = bb.RunTemplate(arrival_rate=1.5, n_requests=4000, batch_size=16, n_servers=2,
                       max_batch_wait=3.0, bins=bb.BinRule(k=4),
                       service=bb.ServiceSpec("uniform", 1.0, 20.0))
    p = bb.run_point(t, 99, 6, rng="reference")
    thr, p99 = [], []
    for r in range(6):
        mr, _ = O.run(O.reference(), dict(arrival_rate=1.5, n_requests=4000, batch_size=16,
                                          n_servers=2, max_batch_wait=3.0,
                                          edges=bb.uniform_boundaries(4, 1.0, 20.0).edges,
                                          lo=1.0, hi=20.0, seed=bb.replication_seed(99, r)),
                      detail=False)
        thr.append(mr["throughput"])
        p99.append(mr["latency_p99"])
    mean = 0.0
    for x in thr:
        mean += x
    mean /= 6
    assert same_bits(p.throughput_mean, mean)
    m99 = 0.0
    for x in p99:
        m99 += x
    assert same_bits(p.latency_p99, m99 / 6)


def test_randomized_timer_runs_match_reference_binary():
    """Random max_batch_wait shapes through run_simulation_detailed with the
    reference's streams: batches, completions and p50/p99 bit-identical."""
    rng = np.random.default_rng(7)
    for trial in range(24):
        k = int(rng.integers(1, 9))
        B = int(rng.choice([1, 2, 5, 16, 33]))
        S = int(rng.choice([1, 1, 2, 4]))
        n = int(rng.integers(max(B, 100), 5000))
        over = rng.random() < 0.2
        lam = math.inf if over else float(bb.throughput(B, k, 1.0, 20.0) * S * rng.uniform(0.3, 1.4))
        flush = bool(rng.random() < 0.6)
        W = float(rng.uniform(0.2, 30.0))
        c = dict(arrival_rate=lam, n_requests=n, batch_size=B, k=k, seed=500 + trial,
                 servers=S, flush=flush, mbw=W)
        if k > 1 and rng.random() < 0.4:
            c["error"] = ("symmetric", float(rng.uniform(0.0, 0.4)))
        ours, ref = configs(c)
        mr, dr = O.run(O.reference(), ref)
        res = bb.run_simulation_detailed(ours)
        r, b = res.requests, res.batches
        ctx = (trial, c)
        assert same_bits(r["completion"], dr["req_completion"]), ctx
        assert same_bits(b["finish_time"], dr["bat_finish"]), ctx
        assert same_bits(b["formed_time"], dr["bat_formed"]), ctx
        assert same_bits(b["members"], dr["members"]), ctx
        for key in ("makespan", "throughput", "latency_p50", "latency_p99"):
            assert same_bits(getattr(res.metrics, key), mr[key]), (key, ctx)
