"""Generated-mode latency quantiles (fused kernel, quantile mode) are exact.

The fused kernel draws every request from Philox counters, so the same
replication can be rebuilt on the host: gaps from the engine's own
exponential variate (bb_exponential_variates), arrivals as the sequential
sum, services from the uniform sampler, error uniforms from the second
stream.  The oracle (C restatement of the reference engine, pinned to the
reference) replays those streams; its p50/p99 -- finish(),
simulator.hpp:289-301 with interpolated_quantile, binning.hpp:97-104 -- must
equal the kernel's per-replication p50/p99 bit for bit."""
import math

import numpy as np
import pytest
import torch

import oracle_py as O
import paper_2412_04504_b200 as bb

pytestmark = pytest.mark.gpu

M32 = np.uint64(0xFFFFFFFF)
PHILOX_M0, PHILOX_M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
PHILOX_W0, PHILOX_W1 = 0x9E3779B9, 0xBB67AE85
KEY0, KEY1 = 0xA4093822, 0x299F31D0


def splitmix64(x):
    m = 2**64 - 1
    x = (x + 0x9E3779B97F4A7C15) & m
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & m
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & m
    return x ^ (x >> 31)


def philox_np(c0, c1, c2, c3):
    n = len(c0)
    x = np.asarray(c0, np.uint64) & M32
    y = np.full(n, c1, np.uint64)
    z = np.full(n, c2, np.uint64)
    w = np.full(n, c3, np.uint64)
    k0, k1 = KEY0, KEY1
    for _ in range(10):
        p0 = PHILOX_M0 * x
        p1 = PHILOX_M1 * z
        x, y, z, w = (((p1 >> np.uint64(32)) ^ y ^ np.uint64(k0)) & M32, p1 & M32,
                      ((p0 >> np.uint64(32)) ^ w ^ np.uint64(k1)) & M32, p0 & M32)
        k0 = (k0 + PHILOX_W0) & 0xFFFFFFFF
        k1 = (k1 + PHILOX_W1) & 0xFFFFFFFF
    return x, y, z, w


def bits53(hi, lo):
    return (hi << np.uint64(21)) | (lo >> np.uint64(11))


def test_numpy_philox_matches_engine():
    for ctr in ([0, 0, 0, 0], [7, 1, 0xDEADBEEF, 0x12345678], [2**32 - 1, 0, 5, 9]):
        ref = bb.philox4x32_10(ctr, [KEY0, KEY1])
        got = philox_np([ctr[0]], ctr[1], ctr[2], ctr[3])
        assert [int(v[0]) for v in got] == ref


def replica_streams(master, r, n, lam, lo, hi, errors):
    sw = splitmix64(bb.replication_seed(master, r))
    c2, c3 = sw & 0xFFFFFFFF, sw >> 32
    i = np.arange(n, dtype=np.uint64)
    rx, ry, rz, rw = philox_np(i, 0, c2, c3)
    xg, xs = bits53(rx, ry), bits53(rz, rw)
    if math.isinf(lam):
        arrivals = np.zeros(n)
    else:
        gaps = bb.exponential_variates(xg, table=True) * (1.0 / lam)
        arrivals = np.cumsum(gaps)  # sequential, like the kernel's clock
    services = lo + (hi - lo) * (xs.astype(np.float64) * 2.0**-53)
    u_err = None
    if errors:
        ex, ey, ez, ew = philox_np(i >> np.uint64(1), 1, c2, c3)
        xe = np.where(i & np.uint64(1), bits53(ez, ew), bits53(ex, ey))
        u_err = xe.astype(np.float64) * 2.0**-53
    return arrivals, services, u_err


def replica_streams_t(t, master, r, errors):
    """The same, with the services from the engine's own sampler for any
    service kind (bb_service_of_keys: the fused kernel's svc_of_key_t)."""
    n, lam = t.n_requests, t.arrival_rate
    sw = splitmix64(bb.replication_seed(master, r))
    c2, c3 = sw & 0xFFFFFFFF, sw >> 32
    i = np.arange(n, dtype=np.uint64)
    rx, ry, rz, rw = philox_np(i, 0, c2, c3)
    xg, xs = bits53(rx, ry), bits53(rz, rw)
    if math.isinf(lam):
        arrivals = np.zeros(n)
    else:
        arrivals = np.cumsum(bb.exponential_variates(xg, table=True) * (1.0 / lam))
    services = bb.service_of_keys(t, xs)
    u_err = None
    if errors:
        ex, ey, ez, ew = philox_np(i >> np.uint64(1), 1, c2, c3)
        xe = np.where(i & np.uint64(1), bits53(ez, ew), bits53(ex, ey))
        u_err = xe.astype(np.float64) * 2.0**-53
    return arrivals, services, u_err


def kernel_rep_metrics(t, reps, master):
    rep = torch.zeros(6 * reps, dtype=torch.float64, device="cuda")
    bb.points_shard_device([t], reps, master, 0, reps, rep.data_ptr())
    torch.cuda.synchronize()
    return rep.view(6, reps).cpu().numpy()


CASES = [
    # (lambda, n, B, k, servers, flush, p_error, max_batch_wait)
    (0.9, 20000, 8, 4, 1, True, 0.0, None),
    (1.3, 30000, 16, 8, 1, True, 0.15, None),
    (0.6, 12000, 4, 1, 1, True, 0.0, None),
    (1.1, 20000, 16, 4, 1, False, 0.0, None),      # no flush: open partials never complete
    (3.0, 20000, 8, 3, 4, True, 0.0, None),        # Kiefer-Wolfowitz dispatch, 4 servers
    (math.inf, 9000, 32, 4, 1, True, 0.0, None),   # overload, drains in bin order
    (math.inf, 9000, 32, 4, 1, False, 0.1, None),  # overload, round-robin rounds
    (math.inf, 6000, 16, 2, 3, True, 0.0, None),   # overload, 3 servers
    (5.0, 777, 8, 16, 1, True, 0.0, None),         # short run, ragged tail
    # max_batch_wait (simulator.hpp:200-201,223-235)
    (0.8, 20000, 16, 4, 1, True, 0.0, 6.0),        # timers and full batches mixed
    (0.5, 15000, 32, 8, 1, False, 0.1, 3.0),       # no flush: the last partials time out too
    (2.0, 20000, 16, 4, 8, True, 0.0, 1.5),        # 8 servers (the reference's timer test shape)
    (0.3, 8000, 8, 1, 1, True, 0.0, 0.5),          # almost every batch formed by its timer
    (math.inf, 9000, 32, 4, 1, False, 0.0, 2.0),   # overload: partials form at W, in arming order
    (math.inf, 9003, 32, 5, 2, False, 0.1, 1e6),   # ... with 2 servers, server idle until W
    (math.inf, 9000, 32, 4, 1, True, 0.0, 2.0),    # overload + flush: the timers go stale
]


@pytest.mark.parametrize("case", CASES)
def test_replication_quantiles_bit_exact(case):
    lam, n, B, k, S, flush, pe, W = case
    lo, hi, master, reps = 1.0, 20.0, 4711, 40
    kw = dict(arrival_rate=lam, n_requests=n, batch_size=B, n_servers=S, flush_partial=flush,
              bins=bb.BinRule(k=k), service=bb.ServiceSpec("uniform", lo, hi), max_batch_wait=W)
    if pe > 0:
        kw["error"] = bb.ErrorSpec("symmetric", pe)
    t = bb.RunTemplate(**kw)
    got = kernel_rep_metrics(t, reps, master)
    edges = bb.uniform_boundaries(k, lo, hi).edges
    for r in (0, 1, 17, reps - 1):
        a, s, u = replica_streams(master, r, n, lam, lo, hi, pe > 0 and k > 1)
        cfg = dict(arrival_rate=lam, n_requests=n, batch_size=B, n_servers=S,
                   flush_partial=flush, edges=edges, lo=lo, hi=hi, service="arrays",
                   error="symmetric" if pe > 0 else "perfect", p_error=pe, max_batch_wait=W)
        m, _ = O.run(O.oracle(), cfg, inputs=dict(arrivals=a, services=s, u_err=u), detail=False)
        assert got[0, r] == pytest.approx(m["throughput"], rel=1e-12), (r, got[:, r], m)
        assert got[2, r] == m["latency_p50"], (r, got[2, r], m["latency_p50"])
        assert got[3, r] == m["latency_p99"], (r, got[3, r], m["latency_p99"])
        # the other metrics: same completions, reassociated sums
        assert got[0, r] == pytest.approx(m["throughput"], rel=1e-12)
        assert got[1, r] == pytest.approx(m["latency_mean"], rel=1e-9)


def test_point_quantile_means_match_reference_statistically():
    lam = 0.95 * bb.throughput(16, 4, 1.0, 20.0)
    t = bb.RunTemplate(arrival_rate=lam, n_requests=20000, batch_size=16, bins=bb.BinRule(k=4),
                       service=bb.ServiceSpec("uniform", 1.0, 20.0))
    reps = 2000
    got = kernel_rep_metrics(t, reps, 99)
    p = bb.run_point(t, 99, reps)
    assert p.latency_p50 == pytest.approx(got[2].mean(), rel=1e-12)
    assert p.latency_p99 == pytest.approx(got[3].mean(), rel=1e-12)
    if not O.have_reference():
        pytest.skip("reference shim not built")
    ms, _ = O.run_replicas(dict(arrival_rate=lam, n_requests=20000, batch_size=16,
                                edges=bb.uniform_boundaries(4, 1.0, 20.0).edges, lo=1.0, hi=20.0),
                           4242, 0, 200, 8)
    for key, row in (("latency_p50", 2), ("latency_p99", 3)):
        ref = np.array([m[key] for m in ms])
        se = math.sqrt(got[row].var(ddof=1) / reps + ref.var(ddof=1) / len(ref))
        assert abs(got[row].mean() - ref.mean()) <= 3.0 * se, key


def test_quantiles_off_leaves_nan_and_same_throughput():
    t = bb.RunTemplate(arrival_rate=1.0, n_requests=5000, batch_size=8, bins=bb.BinRule(k=4),
                       service=bb.ServiceSpec("uniform", 1.0, 20.0))
    on = kernel_rep_metrics(t, 64, 5)
    prev = bb.set_generated_quantiles(False)
    try:
        off = kernel_rep_metrics(t, 64, 5)
    finally:
        bb.set_generated_quantiles(prev)
    assert np.isnan(off[2]).all() and np.isnan(off[3]).all()
    assert np.array_equal(on[[0, 4, 5]], off[[0, 4, 5]])
    # latency_mean: the sum of the latencies themselves vs sum(completions) - sum(arrivals)
    np.testing.assert_allclose(on[1], off[1], rtol=1e-9)
    assert np.isfinite(on[2]).all() and (on[3] >= on[2]).all()


def test_randomized_configs_bit_exact():
    """Random shapes (B = 1 included, timers, servers, overload, errors, no
    flush): every sampled replication's p50/p99 equals the oracle's."""
    rng = np.random.default_rng(20241205)
    for trial in range(40):
        k = int(rng.integers(1, 9))
        B = int(rng.choice([1, 2, 3, 8, 16, 40]))
        S = int(rng.choice([1, 1, 2, 5]))
        n = int(rng.integers(max(B, 200), 6000))
        over = rng.random() < 0.25
        cap = bb.throughput(B, k, 1.0, 20.0) * S
        lam = math.inf if over else float(cap * rng.uniform(0.3, 1.3))
        flush = bool(rng.random() < 0.6)
        W = float(rng.uniform(0.5, 40.0)) if rng.random() < 0.5 else None
        pe = float(rng.choice([0.0, 0.0, 0.2])) if k > 1 else 0.0
        kw = dict(arrival_rate=lam, n_requests=n, batch_size=B, n_servers=S, flush_partial=flush,
                  bins=bb.BinRule(k=k), service=bb.ServiceSpec("uniform", 1.0, 20.0),
                  max_batch_wait=W)
        if pe > 0:
            kw["error"] = bb.ErrorSpec("symmetric", pe)
        reps, master = 8, 1000 + trial
        got = kernel_rep_metrics(bb.RunTemplate(**kw), reps, master)
        edges = bb.uniform_boundaries(k, 1.0, 20.0).edges
        for r in (0, reps - 1):
            a, s, u = replica_streams(master, r, n, lam, 1.0, 20.0, pe > 0)
            cfg = dict(arrival_rate=lam, n_requests=n, batch_size=B, n_servers=S,
                       flush_partial=flush, edges=edges, lo=1.0, hi=20.0, service="arrays",
                       error="symmetric" if pe > 0 else "perfect", p_error=pe, max_batch_wait=W)
            m, _ = O.run(O.oracle(), cfg, inputs=dict(arrivals=a, services=s, u_err=u),
                         detail=False)
            ctx = (trial, r, kw)
            if m["n_completed"] == 0:
                assert got[2, r] == 0.0 and got[3, r] == 0.0, ctx
                continue
            assert got[0, r] == pytest.approx(m["throughput"], rel=1e-12), ctx
            assert got[2, r] == m["latency_p50"], ctx
            assert got[3, r] == m["latency_p99"], ctx


def _cap_linear(B, k, a=0.5, b=0.03, lo=1.0, hi=1024.0):
    return bb.throughput(B, k, a + b * lo, a + b * hi)


SVC_CASES = [
    # (label, service spec, lambda, n, B, k, flush, p_error, reps checked)
    # C3 (BASELINE configs[2]): the benchmarked linear kind at the k=16/B=32 corner
    ("c3_linear_k16_b32", bb.ServiceSpec("linear", 1.0, 1024.0, intercept=0.5, slope=0.03),
     0.9 * _cap_linear(32, 16), 100000, 32, 16, True, 0.0, (0, 33)),
    ("c3_linear_k1_b8_099", bb.ServiceSpec("linear", 1.0, 1024.0, intercept=0.5, slope=0.03),
     0.99 * _cap_linear(8, 1), 100000, 8, 1, True, 0.0, (0, 5)),
    ("linear_errors", bb.ServiceSpec("linear", 1.0, 1024.0, intercept=0.5, slope=0.03),
     0.7 * _cap_linear(16, 8), 30000, 16, 8, True, 0.2, (1, 2)),
    ("exponential_k4", bb.ServiceSpec("exponential", rate=0.1), 0.6 * 16 * 0.1 / 2.0,
     40000, 16, 4, True, 0.0, (0, 7)),
    ("exponential_noflush", bb.ServiceSpec("exponential", rate=1.0), 3.0, 20000, 8, 3, False,
     0.1, (3,)),
    # C5 shape (BASELINE configs[4]): log-normal, k=16, B=64, 10^6-request replications
    ("c5_lognormal_k16_b64", bb.ServiceSpec("lognormal", mu=0.0, sigma=1.0), None,
     1000000, 64, 16, True, 0.0, (0, 1)),
    ("lognormal_overload", bb.ServiceSpec("lognormal", mu=0.0, sigma=1.0), math.inf,
     50000, 64, 16, False, 0.0, (0, 2)),
]


@pytest.mark.parametrize("case", SVC_CASES, ids=[c[0] for c in SVC_CASES])
def test_replication_quantiles_bit_exact_service_kinds(case):
    """p50/p99 bit-exact vs the oracle for the linear (benchmarked), exponential
    and log-normal service kinds, incl. the C3 and C5 corner shapes."""
    _, svc, lam, n, B, k, flush, pe, check = case
    if lam is None:  # 0.9 x the capacity of a pilot overload run
        pilot = bb.run_point(bb.RunTemplate(n_requests=100_000, batch_size=B, bins=bb.BinRule(k=k),
                                            service=svc, flush_partial=False), 7, 64)
        lam = 0.9 * pilot.throughput_mean
    kw = dict(arrival_rate=lam, n_requests=n, batch_size=B, flush_partial=flush,
              bins=bb.BinRule(k=k), service=svc)
    if pe > 0:
        kw["error"] = bb.ErrorSpec("symmetric", pe)
    t = bb.RunTemplate(**kw)
    master = 20241205
    reps = max(check) + 1
    got = kernel_rep_metrics(t, reps, master)
    edges = bb.template_edges(t)
    for r in check:
        a, s, u = replica_streams_t(t, master, r, pe > 0 and k > 1)
        cfg = dict(arrival_rate=lam, n_requests=n, batch_size=B, flush_partial=flush,
                   edges=edges, service="arrays", error="symmetric" if pe > 0 else "perfect",
                   p_error=pe)
        m, _ = O.run(O.oracle(), cfg, inputs=dict(arrivals=a, services=s, u_err=u), detail=False)
        assert m["n_completed"] > 0
        assert got[0, r] == pytest.approx(m["throughput"], rel=1e-12), (r, got[:, r], m)
        assert got[4, r] == m["makespan"], (r, got[4, r], m["makespan"])
        assert got[2, r] == m["latency_p50"], (r, got[2, r], m["latency_p50"])
        assert got[3, r] == m["latency_p99"], (r, got[3, r], m["latency_p99"])
        assert got[1, r] == pytest.approx(m["latency_mean"], rel=1e-9)
