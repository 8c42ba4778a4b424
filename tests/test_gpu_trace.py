"""Trace mode on the B200 vs the reference: bit-exact per-request and
per-batch results (bins, membership, dispatch order, formed/start/finish,
completions, exact p50/p99), through the C ABI (bb_run_trace).

Scalar sums (latency_mean, busy fraction) are compared with the bound of a
reassociated fp64 sum, |ours - ref| <= 2 n 2^-53 sum|x|."""
import math
import random

import numpy as np
import pytest

import oracle_py as O
import paper_2412_04504_b200 as bb
from _helpers import fixture_names, load_fixture, same_bits, sum_tol

pytestmark = pytest.mark.gpu

U64_NONE = np.uint64(2**64 - 1)


def sim_config(cfg):
    em = bb.Perfect()
    if cfg.get("error") == "symmetric":
        em = bb.Symmetric(cfg["p_error"])
    elif cfg.get("error") == "confusion":
        em = bb.Confusion(cfg["confusion"])
    return bb.SimConfig(arrival_rate=cfg["arrival_rate"], n_requests=cfg["n_requests"],
                        batch_size=cfg["batch_size"], bins=bb.BinConfig(list(cfg["edges"])),
                        error_model=em, seed=cfg.get("seed", 0),
                        flush_partial=cfg.get("flush_partial", True))


def check_against(res, exp, n, latency_abs_sum=None):
    """res: bb.SimResult; exp: dict of reference arrays (fixture naming)."""
    r, b = res.requests, res.batches
    assert same_bits(r["true_bin"], exp["req_true_bin"])
    assert same_bits(r["predicted_bin"], exp["req_pred_bin"])
    batch = r["batch"].astype(np.uint64)
    batch[r["batch"] == bb.kNoBatch] = U64_NONE
    assert same_bits(batch, exp["req_batch"])
    assert same_bits(r["completion"], exp["req_completion"])
    assert same_bits(b["bin"], exp["bat_bin"])
    assert same_bits(b["size"], exp["bat_size"])
    assert same_bits(b["first"], exp["bat_first"])
    assert same_bits(b["formed_time"], exp["bat_formed"])
    assert same_bits(b["start_time"], exp["bat_start"])
    assert same_bits(b["finish_time"], exp["bat_finish"])
    assert same_bits(b["service_time"], exp["bat_service"])
    assert same_bits(b["members"], exp["members"])


def check_metrics(m, ref, n, lat_abs, busy_abs):
    assert m.n_completed == ref["n_completed"]
    for key in ("makespan", "throughput", "latency_p50", "latency_p99"):
        assert same_bits(getattr(m, key), ref[key]), key
    assert abs(m.latency_mean - ref["latency_mean"]) <= sum_tol(n, lat_abs) / max(ref["n_completed"], 1)
    if ref["makespan"] > 0:
        assert abs(m.server_busy_fraction - ref["server_busy_fraction"]) <= sum_tol(n, busy_abs) / ref["makespan"]


@pytest.mark.parametrize("name", fixture_names())
def test_golden_fixture_bit_exact(name):
    cfg, metrics, g = load_fixture(name)
    if cfg.get("service") == "trace_cyclic":
        pytest.skip("replay fixture: covered by test_replay_kats")
    u = g["u_err"] if len(g["u_err"]) else None
    res = bb.run_trace(sim_config(cfg), g["arrivals"], g["services"], u_err=u, detailed=True)
    check_against(res, g, cfg["n_requests"])
    lat = g["req_completion"] - g["arrivals"]
    lat_abs = np.nansum(np.abs(lat))
    check_metrics(res.metrics, metrics, cfg["n_requests"], lat_abs, g["bat_service"].sum())
    assert res.metrics.per_bin_batch_counts == list(map(int, g["per_bin"]))


@pytest.mark.parametrize("name", ["kat_1526_k1", "kat_1526_k2", "kat_16_mixed", "kat_16_split"])
def test_replay_kats(name):
    # test_simulator.cpp:293-328 / acceptance.cpp criterion 8: exact makespans
    cfg, metrics, g = load_fixture(name)
    c = sim_config(cfg)
    m = bb.replay_trace(c, cfg["table"])
    assert m.makespan == metrics["makespan"]
    res = bb.replay_trace_detailed(c, cfg["table"])
    check_against(res, g, cfg["n_requests"])


def oracle_case(cfg):
    """Reference-RNG streams + oracle results for a config (oracle = checker)."""
    m, d = O.run(O.oracle(), cfg)
    n = cfg["n_requests"]
    draws = cfg.get("error") == "confusion" or (
        cfg.get("error") == "symmetric" and len(cfg["edges"]) > 2 and cfg.get("p_error", 0) > 0)
    u = O.stream_uniform01(O.oracle(), cfg["seed"], 2, n) if draws else None
    exp = dict(req_true_bin=d["req_true_bin"], req_pred_bin=d["req_pred_bin"],
               req_batch=d["req_batch"], req_completion=d["req_completion"],
               bat_bin=d["bat_bin"], bat_size=d["bat_size"], bat_first=d["bat_first"],
               bat_formed=d["bat_formed"], bat_start=d["bat_start"], bat_finish=d["bat_finish"],
               bat_service=d["bat_service"], members=d["members"])
    return m, d, u, exp


def random_case(seed):
    rng = random.Random(seed)
    k = rng.choice([1, 2, 3, 5, 8, 16, 32])
    B = rng.choice([1, 2, 3, 8, 16, 64, 128])
    n = rng.randint(B, rng.choice([500, 5000, 60000]))
    cap = bb.throughput(B, k, 1.0, 20.0)
    lam = math.inf if rng.random() < 0.25 else cap * rng.choice([0.3, 0.7, 0.95, 0.99, 1.2])
    cfg = dict(arrival_rate=lam, n_requests=n, batch_size=B,
               edges=bb.uniform_boundaries(k, 1.0, 20.0).edges, lo=1.0, hi=20.0,
               seed=rng.getrandbits(64), flush_partial=rng.random() < 0.7)
    e = rng.choice(["perfect", "symmetric", "confusion"])
    if e == "symmetric":
        cfg.update(error="symmetric", p_error=rng.choice([0.0, 0.1, 0.5]))
    elif e == "confusion":
        w = np.random.default_rng(seed).random((k, k)) + 0.05
        cfg.update(error="confusion", confusion=(w / w.sum(1, keepdims=True)).tolist())
    return cfg


@pytest.mark.parametrize("seed", range(40))
def test_random_configs_bit_exact(seed):
    cfg = random_case(seed)
    m, d, u, exp = oracle_case(cfg)
    res = bb.run_trace(sim_config(cfg), d["req_arrival"], d["req_service"], u_err=u, detailed=True)
    check_against(res, exp, cfg["n_requests"])
    lat = d["req_completion"] - d["req_arrival"]
    check_metrics(res.metrics, m, cfg["n_requests"], np.nansum(np.abs(lat)),
                  d["bat_service"].sum())


def test_pred_bin_input_overrides_error_model():
    cfg = random_case(3)
    cfg.update(error="symmetric", p_error=0.3, edges=bb.uniform_boundaries(4, 1.0, 20.0).edges)
    m, d, u, exp = oracle_case(cfg)
    res = bb.run_trace(sim_config(dict(cfg, error="perfect")), d["req_arrival"], d["req_service"],
                       pred_bin=d["req_pred_bin"].astype(np.uint8), detailed=True)
    check_against(res, exp, cfg["n_requests"])


def test_small_tie_groups_use_fast_path_exactly():
    # quantised arrivals: tie groups of size <= B follow closing-index order
    rng = np.random.default_rng(5)
    n, B, k = 20000, 16, 4
    a = np.floor(np.cumsum(rng.exponential(1 / 3.0, n)) * 4) / 4  # many ties
    s = rng.uniform(1.0, 20.0, n)
    edges = bb.uniform_boundaries(k, 1.0, 20.0).edges
    cfg = dict(arrival_rate=3.0, n_requests=n, batch_size=B, edges=edges, seed=0, service="arrays")
    m, d = O.run(O.oracle(), cfg, dict(arrivals=a, services=s))
    res = bb.run_trace(sim_config(cfg), a, s, detailed=True)
    check_against(res, {key: d[key] for key in d}, n)


def _tie_case(seed):
    """given arrivals with tie groups of more than B equal times at finite
    times (App. A.2 rules 1-3), incl. a final group larger than B"""
    rng = np.random.default_rng(77 + seed)
    r = random.Random(seed)
    k = r.choice([1, 2, 3, 4, 8, 16])
    B = r.choice([1, 2, 4, 8, 16])
    n = r.randint(2000, 40000)
    a = np.floor(np.cumsum(rng.exponential(1.0 / r.uniform(0.5, 4.0), n)) / r.choice([1.0, 4.0, 16.0]))
    for _ in range(r.randint(1, 6)):
        i = int(rng.integers(0, n - 1))
        a[i:i + r.randint(B + 1, 8 * B + 3)] = a[i]
    if r.random() < 0.4:
        a[-r.randint(B + 1, 6 * B + 1):] = a[-1]
    a = np.maximum.accumulate(a)
    s = rng.uniform(1.0, 20.0, n)
    cfg = dict(arrival_rate=2.0, n_requests=n, batch_size=B, seed=r.getrandbits(64),
               edges=bb.uniform_boundaries(k, 1.0, 20.0).edges, service="arrays",
               flush_partial=r.random() < 0.6, n_servers=r.choice([1, 1, 1, 3]))
    if r.random() < 0.5:
        cfg.update(error="symmetric", p_error=r.choice([0.1, 0.4]))
    return cfg, a, s


@pytest.mark.parametrize("seed", range(16))
def test_large_tie_groups_bit_exact(seed):
    """Tie groups larger than B at finite times: round-robin formations in
    first-closing order, drains in bin order in the final group -- bit-exact
    against the reference's own event loop on the same arrays (bbref_run_arrays;
    the C restatement where the reference shim is not built)."""
    cfg, a, s = _tie_case(seed)
    n = cfg["n_requests"]
    g = np.diff(np.flatnonzero(np.r_[True, np.diff(a) != 0, True]))
    assert g.max() > cfg["batch_size"]  # the case exercises the general path
    draws = cfg.get("error") == "symmetric" and len(cfg["edges"]) > 2
    u = O.stream_uniform01(O.oracle(), cfg["seed"], 2, n) if draws else None
    lib = O.reference() if O.have_reference() else O.oracle()
    m, d = O.run(lib, cfg, dict(arrivals=a, services=s) if lib is O.reference()
                 else dict(arrivals=a, services=s, u_err=u))
    c = sim_config(cfg)
    c.n_servers = cfg["n_servers"]
    res = bb.run_trace(c, a, s, u_err=u, detailed=True)
    check_against(res, {key: d[key] for key in d}, n)
    lat = d["req_completion"] - d["req_arrival"]
    check_metrics(res.metrics, m, n, np.nansum(np.abs(lat)), d["bat_service"].sum())


def test_errors_have_reference_categories():
    n, B = 64, 4
    a = np.arange(n, dtype=np.float64)
    s = np.full(n, 5.0)
    c = sim_config(dict(arrival_rate=1.0, n_requests=n, batch_size=B, edges=[1.0, 10.0, 20.0]))
    s_bad = s.copy()
    s_bad[17] = 50.0
    with pytest.raises(bb.DomainError):  # binning.hpp:135-140
        bb.run_trace(c, a, s_bad)
    s_bad[17] = -1.0
    with pytest.raises(bb.DomainError):  # simulator.hpp:189-190
        bb.run_trace(c, a, s_bad)
    a_bad = a.copy()
    a_bad[30] = 1.0
    with pytest.raises(bb.InvalidArgument):
        bb.run_trace(c, a_bad, s)
    p = np.ones(n, np.uint8)
    p[3] = 9
    with pytest.raises(bb.InvalidArgument):
        bb.run_trace(c, a, s, pred_bin=p)


def test_full_size_c2_trace_bit_exact():
    """BASELINE config 2 at full size: 10^7 requests, k=8, B=16, from the
    reference generator (restated by the oracle, pinned bit-for-bit)."""
    cfg = dict(arrival_rate=0.95 * 1.385550, n_requests=10_000_000, batch_size=16,
               edges=bb.uniform_boundaries(8, 1.0, 20.0).edges, lo=1.0, hi=20.0, seed=1001,
               error="symmetric", p_error=0.1)
    m, d, u, exp = oracle_case(cfg)
    res = bb.run_trace(sim_config(cfg), d["req_arrival"], d["req_service"], u_err=u, detailed=True)
    check_against(res, exp, cfg["n_requests"])
    lat = d["req_completion"] - d["req_arrival"]
    check_metrics(res.metrics, m, cfg["n_requests"], np.nansum(np.abs(lat)), d["bat_service"].sum())


@pytest.mark.parametrize("servers,load", [(4, 0.5), (4, 1.3), (64, 0.6), (3, 0.99)])
def test_multi_server_chunk_parallel_dispatch_bit_exact(servers, load):
    """Kiefer-Wolfowitz dispatch over ~1e5 batches (chunks of 1024 dispatched
    from an all-idle state, re-dispatched serially where a server is still
    busy at the chunk's first formation): start/finish, completions and the
    busy fraction (the sequential busy-time sum) bit-identical to the oracle,
    in light load (most chunks speculative) and overload (all re-dispatched)."""
    n, B, k = 1_600_000, 16, 4
    cap = servers * bb.throughput(B, k, 1.0, 20.0)
    cfg = dict(arrival_rate=load * cap, n_requests=n, batch_size=B,
               edges=bb.uniform_boundaries(k, 1.0, 20.0).edges, lo=1.0, hi=20.0, seed=4242 + servers,
               n_servers=servers)
    m, d, u, exp = oracle_case(cfg)
    c = sim_config(cfg)
    c.n_servers = servers
    res = bb.run_trace(c, d["req_arrival"], d["req_service"], detailed=True)
    check_against(res, exp, n)
    assert same_bits(res.metrics.makespan, m["makespan"])
    assert same_bits(res.metrics.server_busy_fraction, m["server_busy_fraction"])
    assert same_bits(res.metrics.latency_p99, m["latency_p99"])
