"""Generated mode (Philox, fused per-replication kernel) vs the reference:
point means within 3 standard errors of the reference's own replications
(BASELINE configs 1, 3, 4, 5 shapes), the paper's closed-form k-bin
throughput at overload (Theorem 1, 2%), and consistency with the
single-run pipeline on the same Philox streams."""
import math

import numpy as np
import pytest
import torch

import oracle_py as O
import paper_2412_04504_b200 as bb

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.have_reference(), reason="reference shim not built")]

THREADS = 8


def ref_stats(cfg, reps, master=4242):
    ms, _ = O.run_replicas(cfg, master, 0, reps, THREADS)
    thr = np.array([m["throughput"] for m in ms])
    lat = np.array([m["latency_mean"] for m in ms])
    return thr, lat


def within_3se(gpu_mean, gpu_std, gpu_n, ref):
    se = math.sqrt(gpu_std**2 / gpu_n + ref.std(ddof=1) ** 2 / len(ref))
    return abs(gpu_mean - ref.mean()) <= 3.0 * se + 1e-12 * abs(ref.mean())


def template(**kw):
    svc = kw.pop("service", bb.ServiceSpec("uniform", 1.0, 20.0))
    return bb.RunTemplate(service=svc, **kw)


@pytest.mark.parametrize("k", [1, 4])
def test_c1_uniform_near_capacity(k):
    lam = 0.95 * bb.throughput(4, k, 1.0, 20.0)
    t = template(arrival_rate=lam, n_requests=10_000, batch_size=4, bins=bb.BinRule(k=k))
    p = bb.run_point(t, 1001, 4000)
    thr, lat = ref_stats(dict(arrival_rate=lam, n_requests=10_000, batch_size=4,
                              edges=bb.uniform_boundaries(k, 1.0, 20.0).edges, lo=1.0, hi=20.0), 400)
    assert within_3se(p.throughput_mean, p.throughput_std, 4000, thr)
    assert within_3se(p.latency_mean, p.latency_std, 4000, lat)


def test_c3_linear_service_point():
    a, b = 0.5, 0.03
    lo, hi = b * 1 + a, b * 1024 + a
    lam = 0.9 * bb.throughput(32, 8, lo, hi)
    svc = bb.ServiceSpec("linear", 1.0, 1024.0, intercept=a, slope=b)
    t = template(arrival_rate=lam, n_requests=100_000, batch_size=32, bins=bb.BinRule(k=8),
                 service=svc)
    p = bb.run_point(t, 7, 2000)
    thr, lat = ref_stats(dict(arrival_rate=lam, n_requests=100_000, batch_size=32,
                              edges=bb.uniform_boundaries(8, lo, hi).edges, service="linear",
                              lo=1.0, hi=1024.0, lin_a=a, lin_b=b), 48)
    assert within_3se(p.throughput_mean, p.throughput_std, 2000, thr)
    assert within_3se(p.latency_mean, p.latency_std, 2000, lat)
    assert p.analytic_latency == pytest.approx(bb.expected_latency(32, 8, lo, hi, lam))


@pytest.mark.parametrize("pe", [0.0, 0.15, 0.3])
def test_c4_symmetric_errors(pe):
    lam = 0.9 * bb.throughput(32, 8, 1.0, 20.0)
    t = template(arrival_rate=lam, n_requests=100_000, batch_size=32, bins=bb.BinRule(k=8),
                 error=bb.ErrorSpec("symmetric", pe))
    p = bb.run_point(t, 11, 2000)
    thr, lat = ref_stats(dict(arrival_rate=lam, n_requests=100_000, batch_size=32,
                              edges=bb.uniform_boundaries(8, 1.0, 20.0).edges, lo=1.0, hi=20.0,
                              error="symmetric", p_error=pe), 48)
    assert within_3se(p.throughput_mean, p.throughput_std, 2000, thr)
    assert within_3se(p.latency_mean, p.latency_std, 2000, lat)


C4_PE = [0.0, 0.05, 0.10, 0.15, 0.20, 0.25, 0.30]


@pytest.mark.parametrize("k", [4, 8])
@pytest.mark.parametrize("overload", [False, True], ids=["lam0.9cap", "overload"])
def test_c4_full_grid_3se_and_monotone(k, overload):
    """BASELINE configs[3]: k in {4, 8}, B=32, U[1,20], symmetric p_e 0..0.30,
    at 0.9 x capacity and at overload.  Every point within 3 SE of the
    reference's own replications; with common random numbers across p_e
    (the error stream is separate, binning.hpp:239-240) overload throughput
    is non-increasing and finite-rate latency non-decreasing in p_e."""
    lam = math.inf if overload else 0.9 * bb.throughput(32, k, 1.0, 20.0)
    n = 100_000
    base = template(arrival_rate=lam, n_requests=n, batch_size=32, bins=bb.BinRule(k=k))
    reps = 2000
    pts = bb.run_experiment(bb.ExperimentSpec(base=base, axes=[bb.SweepAxis("p_e", C4_PE)],
                                              replications=reps, seed=4))
    assert [p.p_error for p in pts] == C4_PE
    edges = bb.uniform_boundaries(k, 1.0, 20.0).edges
    for p in pts:
        thr, lat = ref_stats(dict(arrival_rate=lam, n_requests=n, batch_size=32, edges=edges,
                                  lo=1.0, hi=20.0, error="symmetric", p_error=p.p_error), 32)
        assert within_3se(p.throughput_mean, p.throughput_std, reps, thr), p
        assert within_3se(p.latency_mean, p.latency_std, reps, lat), p
    for a, b in zip(pts, pts[1:]):
        if overload:
            assert b.throughput_mean <= a.throughput_mean, (a.p_error, b.p_error)
        else:
            assert b.latency_mean >= a.latency_mean, (a.p_error, b.p_error)
    if overload:  # p_e = 0 reproduces Theorem 1 (2%)
        pred = bb.throughput(32, k, 1.0, 20.0)
        assert abs(pts[0].throughput_mean - pred) / pred < 0.02


def test_c5_lognormal_overload():
    t = template(arrival_rate=bb.kOverload, n_requests=100_000, batch_size=64,
                 bins=bb.BinRule(k=16), service=bb.ServiceSpec("lognormal", mu=0.0, sigma=1.0))
    p = bb.run_point(t, 5, 1000)
    edges = None
    # the same host-computed quantile edges the engine materialises
    import paper_2412_04504_b200._capi  # noqa
    from scipy.stats import norm
    edges = [0.0] + [math.exp(norm.ppf(j / 16)) for j in range(1, 16)] + [math.inf]
    thr, lat = ref_stats(dict(arrival_rate=math.inf, n_requests=100_000, batch_size=64,
                              edges=edges, service="lognormal", mu=0.0, sigma=1.0), 48)
    assert within_3se(p.throughput_mean, p.throughput_std, 1000, thr)
    assert within_3se(p.latency_mean, p.latency_std, 1000, lat)


def test_theorem1_overload_capacity_and_reference():
    # acceptance criterion 1: B=128, U[1,20], overload, no flush, k=1..5
    base = template(n_requests=12800, batch_size=128, flush_partial=False)
    spec = bb.ExperimentSpec(base=base, axes=[bb.SweepAxis("k", [1, 2, 3, 5])], replications=400,
                             seed=1001)
    prev = 0.0
    for p in bb.run_experiment(spec):
        pred = bb.throughput(128, p.k, 1.0, 20.0)
        assert abs(p.throughput_mean - pred) / pred < 0.02
        assert p.analytic_throughput == pytest.approx(pred)
        assert p.throughput_mean > prev
        prev = p.throughput_mean
        thr, lat = ref_stats(dict(arrival_rate=math.inf, n_requests=12800, batch_size=128,
                                  edges=bb.uniform_boundaries(p.k, 1.0, 20.0).edges, lo=1.0,
                                  hi=20.0, flush_partial=False), 200)
        assert within_3se(p.throughput_mean, p.throughput_std, 400, thr)
        assert within_3se(p.latency_mean, p.latency_std, 400, lat)


def test_overload_with_flush_and_errors_vs_reference():
    base = template(n_requests=3003, batch_size=16, flush_partial=True, bins=bb.BinRule(k=5),
                    error=bb.ErrorSpec("symmetric", 0.2))
    p = bb.run_point(base, 3, 4000)
    thr, lat = ref_stats(dict(arrival_rate=math.inf, n_requests=3003, batch_size=16,
                              edges=bb.uniform_boundaries(5, 1.0, 20.0).edges, lo=1.0, hi=20.0,
                              error="symmetric", p_error=0.2), 800)
    assert within_3se(p.throughput_mean, p.throughput_std, 4000, thr)
    assert within_3se(p.latency_mean, p.latency_std, 4000, lat)


def test_poisson_no_flush_vs_reference():
    t = template(arrival_rate=0.8, n_requests=5000, batch_size=16, flush_partial=False,
                 bins=bb.BinRule(k=3))
    p = bb.run_point(t, 9, 4000)
    thr, lat = ref_stats(dict(arrival_rate=0.8, n_requests=5000, batch_size=16,
                              edges=bb.uniform_boundaries(3, 1.0, 20.0).edges, lo=1.0, hi=20.0,
                              flush_partial=False), 800)
    assert within_3se(p.throughput_mean, p.throughput_std, 4000, thr)
    assert within_3se(p.latency_mean, p.latency_std, 4000, lat)


def test_confusion_and_exponential_vs_reference():
    rows = [[0.7, 0.25, 0.05], [0.15, 0.7, 0.15], [0.02, 0.28, 0.7]]
    t = template(arrival_rate=0.5, n_requests=4000, batch_size=8, bins=bb.BinRule(k=3),
                 service=bb.ServiceSpec("exponential", rate=0.2),
                 error=bb.ErrorSpec("confusion", rows=rows))
    p = bb.run_point(t, 13, 4000)
    edges = bb.exponential_boundaries(3, 0.2, 8).edges
    thr, lat = ref_stats(dict(arrival_rate=0.5, n_requests=4000, batch_size=8, edges=edges,
                              service="exponential", rate=0.2, error="confusion",
                              confusion=rows), 800)
    assert within_3se(p.throughput_mean, p.throughput_std, 4000, thr)
    assert within_3se(p.latency_mean, p.latency_std, 4000, lat)


def test_trace_replay_generated_monotone_in_k():
    # acceptance criterion 10: Pareto-like trace, B=32, overload, resample
    trace = O.acceptance_trace().tolist()  # acceptance.cpp:366-375, the reference's own trace
    base = bb.RunTemplate(n_requests=12800, batch_size=32, flush_partial=False,
                          service=bb.ServiceSpec("trace", trace_times=trace, trace_mode="resample"))
    spec = bb.ExperimentSpec(base=base, axes=[bb.SweepAxis("k", [1, 2, 4, 8, 16, 32])],
                             replications=200, seed=1001)
    pts = bb.run_experiment(spec)
    thr = [p.throughput_mean for p in pts]
    assert all(b >= a * (1 - 1e-9) for a, b in zip(thr, thr[1:]))
    # 3 standard errors against the reference's own replications (the
    # published 10-replication curve, proj/test_output.txt:26, is itself
    # noisy for this heavy-tailed trace; its exact reproduction is checked
    # bit-for-bit in test_gpu_reference_rng.py)
    for p in pts:
        if p.k not in (1, 8, 32):
            continue
        edges = bb.empirical_boundaries(p.k, trace).edges
        ref, _ = ref_stats(dict(arrival_rate=math.inf, n_requests=12800, batch_size=32,
                                edges=edges, flush_partial=False, service="trace_resample",
                                table=trace), 400)
        assert within_3se(p.throughput_mean, p.throughput_std, 200, ref)


def test_fused_replica_equals_single_run_on_same_streams():
    t = template(arrival_rate=1.2, n_requests=20000, batch_size=16, bins=bb.BinRule(k=8))
    p = bb.run_point(t, 77, 1)
    cfg = bb.SimConfig(arrival_rate=1.2, n_requests=20000, batch_size=16,
                       bins=bb.uniform_boundaries(8, 1.0, 20.0), service=bb.Uniform(1.0, 20.0),
                       seed=bb.replication_seed(77, 0))
    m = bb.run_simulation(cfg)
    assert m.throughput == pytest.approx(p.throughput_mean, rel=1e-9)
    assert m.latency_mean == pytest.approx(p.latency_mean, rel=1e-9)


def test_results_independent_of_shards():
    t = template(arrival_rate=1.0, n_requests=5000, batch_size=8, bins=bb.BinRule(k=4))
    spec = bb.ExperimentSpec(base=t, axes=[bb.SweepAxis("lambda", [0.5, 1.0])], replications=96,
                             seed=3)
    whole = bb.run_experiment(spec)
    import torch
    P = bb.experiment_points(spec)
    rep = torch.zeros(6 * P * 96, dtype=torch.float64, device="cuda")
    for lo, hi in ((0, 40), (40, 41), (41, 96)):
        bb.sweep_shard_device(spec, lo, hi, rep.data_ptr())
    torch.cuda.synchronize()
    pts = bb.sweep_reduce_device(spec, rep.data_ptr())
    for a, b in zip(whole, pts):
        assert a.throughput_mean == b.throughput_mean and a.latency_std == b.latency_std


# ---------------------------------------------------------------- multi-server
@pytest.mark.parametrize("S,lam,k", [(2, 5.0, 3), (4, 3.0, 2), (64, 5.0, 1)])
def test_multi_server_vs_reference(S, lam, k):
    # test_simulator.cpp:60-83 (2 servers), acceptance.cpp criterion 3 (64 servers)
    B, n = (16, 1003) if S < 64 else (128, 12800)
    t = template(arrival_rate=lam, n_requests=n, batch_size=B, n_servers=S, bins=bb.BinRule(k=k))
    p = bb.run_point(t, 21, 2000)
    thr, lat = ref_stats(dict(arrival_rate=lam, n_requests=n, batch_size=B, n_servers=S,
                              edges=bb.uniform_boundaries(k, 1.0, 20.0).edges, lo=1.0, hi=20.0),
                         200 if S < 64 else 40)
    assert within_3se(p.throughput_mean, p.throughput_std, 2000, thr)
    assert within_3se(p.latency_mean, p.latency_std, 2000, lat)


def test_acceptance_criterion3_latency_formula():
    # acceptance.cpp:126-165: 64 servers, B=128, U[1,20], lambda in {5,10}, k=1..3, within 5%
    base = template(n_requests=12800, batch_size=128, n_servers=64)
    spec = bb.ExperimentSpec(base=base, axes=[bb.SweepAxis("lambda", [5.0, 10.0]),
                                              bb.SweepAxis("k", [1, 2, 3])],
                             replications=10, seed=1001)
    for p in bb.run_experiment(spec):
        pred = bb.expected_latency(128, p.k, 1.0, 20.0, p.arrival_rate)
        assert abs(p.latency_mean - pred) / pred < 0.05
        assert p.analytic_latency == pytest.approx(pred)


@pytest.mark.parametrize("S,k,flush", [(2, 3, True), (8, 4, False), (64, 2, True)])
def test_multi_server_overload_vs_reference(S, k, flush):
    # overload with S servers (paper Fig. 6: 8 servers): batches in dispatch
    # order through the Kiefer-Wolfowitz recursion; 3-sigma vs the reference
    B, n = 16, 2003
    t = template(n_requests=n, batch_size=B, n_servers=S, flush_partial=flush,
                 bins=bb.BinRule(k=k))
    p = bb.run_point(t, 33, 2000)
    thr, lat = ref_stats(dict(arrival_rate=math.inf, n_requests=n, batch_size=B, n_servers=S,
                              flush_partial=flush,
                              edges=bb.uniform_boundaries(k, 1.0, 20.0).edges, lo=1.0, hi=20.0),
                         200)
    assert within_3se(p.throughput_mean, p.throughput_std, 2000, thr)
    assert within_3se(p.latency_mean, p.latency_std, 2000, lat)


# ------------------------------------------------------------- max_batch_wait
@pytest.mark.parametrize("W,flush,S", [(4.0, True, 1), (2.0, False, 1), (1.5, True, 8)])
def test_max_batch_wait_vs_reference(W, flush, S):
    """Timers (simulator.hpp:200-201,223-235) in the fused kernel: point means
    (throughput, latency, p50) within 3 SE of the reference's own replications.
    (Short waits form small batches: the queue can then overload, as in the
    reference.)"""
    lam = 0.6 * S
    base = dict(arrival_rate=lam, n_requests=10_000, batch_size=16, n_servers=S,
                flush_partial=flush)
    t = template(bins=bb.BinRule(k=4), max_batch_wait=W, **base)
    p = bb.run_point(t, 31, 2000)
    ms, _ = O.run_replicas(dict(base, edges=bb.uniform_boundaries(4, 1.0, 20.0).edges, lo=1.0,
                                hi=20.0, max_batch_wait=W), 4242, 0, 300, THREADS)
    thr = np.array([m["throughput"] for m in ms])
    lat = np.array([m["latency_mean"] for m in ms])
    assert within_3se(p.throughput_mean, p.throughput_std, 2000, thr)
    assert within_3se(p.latency_mean, p.latency_std, 2000, lat)
    p50 = np.array([m["latency_p50"] for m in ms])
    rep = torch.zeros(6 * 2000, dtype=torch.float64, device="cuda")
    bb.points_shard_device([t], 2000, 31, 0, 2000, rep.data_ptr())
    torch.cuda.synchronize()
    g50 = rep.view(6, 2000)[2].cpu().numpy()
    assert g50.mean() == pytest.approx(p.latency_p50, rel=1e-12)
    assert within_3se(g50.mean(), g50.std(ddof=1), 2000, p50)
