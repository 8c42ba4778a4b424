"""run_point / run_experiment with the reference's own random streams
(rng="reference") against the reference binary's run_point
(experiment.hpp:254-307), every PointResult field.

Per replication the engine reproduces the reference's SimResult (trace
pipeline on the reference streams); the per-point reduction is mean_std
(experiment.hpp:188-200) in replication order with no FMA contraction.  So
throughput mean/std, p50/p99 means, makespan and the analytic columns are
bit-identical; latency_mean/std and the busy fraction inherit the
reassociation bound of the per-replication latency and busy sums."""
import math

import pytest

import oracle_py as O
import paper_2412_04504_b200 as bb
from _helpers import same_bits

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.have_reference(), reason="reference shim not built")]

EXACT = ("throughput_mean", "throughput_std", "latency_p50", "latency_p99", "makespan_mean",
         "analytic_throughput", "analytic_latency", "analytic_max_throughput")
CLOSE = ("latency_mean", "latency_std", "busy_fraction_mean")

CONF3 = [[0.7, 0.25, 0.05], [0.15, 0.7, 0.15], [0.02, 0.28, 0.7]]

CASES = [
    # acceptance criterion 1/2 protocol (overload, no flush), k = 2
    dict(lam=math.inf, n=12800, B=128, k=2, flush=False),
    # finite rate, symmetric errors, 2 servers (criterion 9 shape, several reps)
    dict(lam=7.0, n=997, B=13, k=3, servers=2, err=("symmetric", 0.15)),
    # C1 shape: k=4, B=4, 0.95 x capacity
    dict(lam=0.95 * 0.3186594, n=10000, B=4, k=4),
    # exponential service, derived open-ended edges, flush
    dict(lam=0.5, n=6000, B=8, k=3, svc=("exponential", 0.2)),
    # confusion-matrix errors
    dict(lam=3.0, n=4000, B=8, k=3, err=("confusion", CONF3)),
    # trace service (resample, the ServiceSpec default), empirical edges
    dict(lam=math.inf, n=12800, B=32, k=4, svc=("trace", "resample"), flush=False),
    # timers + 3 servers
    dict(lam=2.5, n=8000, B=8, k=3, servers=3, mbw=0.75),
]


def _both(c, trace):
    svc = c.get("svc", ("uniform",))
    ref = dict(arrival_rate=c["lam"], n_requests=c["n"], batch_size=c["B"],
               n_servers=c.get("servers", 1), flush_partial=c.get("flush", True),
               max_batch_wait=c.get("mbw"))
    if svc[0] == "uniform":
        spec = bb.ServiceSpec("uniform", 1.0, 20.0)
        ref.update(service="uniform", lo=1.0, hi=20.0)
    elif svc[0] == "exponential":
        spec = bb.ServiceSpec("exponential", rate=svc[1])
        ref.update(service="exponential", rate=svc[1])
    else:
        spec = bb.ServiceSpec("trace", trace_times=list(trace), trace_mode=svc[1])
        ref.update(service="trace_" + svc[1], table=trace)
    err = bb.ErrorSpec()
    if "err" in c:
        kind, p = c["err"]
        if kind == "symmetric":
            err = bb.ErrorSpec("symmetric", p)
            ref.update(error="symmetric", p_error=p)
        else:
            err = bb.ErrorSpec("confusion", rows=p)
            ref.update(error="confusion", confusion=p)
    t = bb.RunTemplate(arrival_rate=c["lam"], n_requests=c["n"], batch_size=c["B"],
                       n_servers=c.get("servers", 1), flush_partial=c.get("flush", True),
                       max_batch_wait=c.get("mbw"), service=spec, bins=bb.BinRule(k=c["k"]),
                       error=err)
    return t, ref


@pytest.mark.parametrize("i", range(len(CASES)))
def test_run_point_every_field_matches_reference(i):
    c = CASES[i]
    trace = O.acceptance_trace(20000)
    t, ref = _both(c, trace)
    reps, master = 6, 1001 + i
    got = bb.run_point(t, master, reps, rng="reference")
    want = O.run_point(ref, c["k"], master, reps)
    for f in EXACT:
        g, w = getattr(got, f), want[f]
        assert same_bits(g, w) or (math.isnan(g) and math.isnan(w)), (f, g, w)
    for f in CLOSE:
        assert getattr(got, f) == pytest.approx(want[f], rel=1e-12, abs=1e-12), f
    assert got.k == c["k"] and got.replications == reps and got.n_requests == c["n"]


def test_run_experiment_sweep_std_matches_reference():
    """A k x p_e sweep (criterion 7 shape, smaller): throughput_std of every
    point bit-identical to the reference's run_point over the same seeds."""
    base = bb.RunTemplate(n_requests=3200, batch_size=32, flush_partial=False,
                          service=bb.ServiceSpec("uniform", 1.0, 20.0))
    spec = bb.ExperimentSpec(base=base, axes=[bb.SweepAxis("k", [2, 4]),
                                              bb.SweepAxis("p_e", [0.0, 0.1, 0.25])],
                             replications=5, seed=1001, rng="reference")
    for p in bb.run_experiment(spec):
        ref = dict(arrival_rate=math.inf, n_requests=3200, batch_size=32, flush_partial=False,
                   lo=1.0, hi=20.0, error="symmetric", p_error=p.p_error)
        w = O.run_point(ref, p.k, 1001, 5)
        assert same_bits(p.throughput_mean, w["throughput_mean"]), (p.k, p.p_error)
        assert same_bits(p.throughput_std, w["throughput_std"]), (p.k, p.p_error)
        assert same_bits(p.latency_p99, w["latency_p99"]), (p.k, p.p_error)
