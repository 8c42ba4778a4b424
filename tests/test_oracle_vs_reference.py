"""Randomised bit-for-bit agreement of the C restatement with the reference
engine itself (oracle/_ref/libbbref.so) across the SimConfig space."""
import math
import random

import numpy as np
import pytest

import oracle_py as O
from _helpers import BAT_KEYS, REQ_KEYS, same_bits

pytestmark = pytest.mark.skipif(not O.have_reference(), reason="reference shim not built")


def random_config(rng: random.Random):
    k = rng.choice([1, 2, 3, 4, 8, 16])
    B = rng.choice([1, 2, 4, 8, 16, 32])
    n = rng.randint(B, 3000)
    svc = rng.choice(["uniform", "uniform", "exponential", "trace_cyclic", "trace_resample",
                      "empirical", "linear", "lognormal"])
    cfg = dict(n_requests=n, batch_size=B, seed=rng.getrandbits(64),
               flush_partial=rng.random() < 0.7, n_servers=rng.choice([1, 1, 1, 2, 3]))
    cfg["arrival_rate"] = math.inf if rng.random() < 0.3 else rng.uniform(0.05, 3.0)
    if svc in ("uniform", "linear"):
        lo, hi = 1.0, 20.0
        cfg.update(lo=lo, hi=hi)
        if svc == "linear":
            cfg.update(lo=1.0, hi=1024.0, lin_a=0.5, lin_b=0.03)
            lo, hi = 0.53, 0.5 + 0.03 * 1024
        cfg["edges"] = O.uniform_boundaries(k, lo, hi).tolist()
    elif svc in ("exponential", "lognormal"):
        cfg.update(rate=0.3, mu=0.0, sigma=1.0)
        cfg["edges"] = [0.0] + sorted(rng.uniform(0.1, 8.0) for _ in range(k - 1)) + [math.inf]
        if len(set(cfg["edges"])) != len(cfg["edges"]):
            cfg["edges"] = [0.0] + [0.5 * (j + 1) for j in range(k - 1)] + [math.inf]
    else:
        table = [rng.choice([1.0, 2.0, 3.5, 5.0, 7.25, 9.0, 12.0, 20.0]) for _ in range(rng.randint(4, 50))]
        cfg["table"] = table
        cfg["edges"] = [1.0] + [1.0 + 19.0 * (j + 1) / k for j in range(k - 1)] + [20.0]
    cfg["service"] = svc
    err = rng.choice(["perfect", "symmetric", "confusion"])
    cfg["error"] = err
    if err == "symmetric":
        cfg["p_error"] = rng.choice([0.0, 0.05, 0.3, 0.5])
    elif err == "confusion":
        rows = []
        for _ in range(k):
            w = np.array([rng.random() for _ in range(k)])
            rows.append((w / w.sum()).tolist())
        cfg["confusion"] = rows
    if rng.random() < 0.15:
        cfg["max_batch_wait"] = rng.uniform(0.5, 5.0)
    return cfg


@pytest.mark.parametrize("seed", range(60))
def test_oracle_equals_reference(seed):
    cfg = random_config(random.Random(seed))
    try:
        mr, dr = O.run(O.reference(), cfg)
    except O.OracleError as e:
        with pytest.raises(O.OracleError) as ei:
            O.run(O.oracle(), cfg)
        assert ei.value.code == e.code
        return
    mo, do = O.run(O.oracle(), cfg)
    for key in REQ_KEYS + BAT_KEYS + ("req_arrival", "req_service", "members",
                                      "per_bin_batch_counts"):
        assert same_bits(do[key], dr[key]), key
    for key in ("throughput", "makespan", "latency_mean", "latency_p50", "latency_p99",
                "server_busy_fraction", "n_completed", "n_batches"):
        assert same_bits(mo[key], mr[key]), key


def tied_arrivals(rng: np.random.Generator, n, rate, quantum, bursts=0, burst_len=0):
    """non-decreasing arrivals with tie groups: Poisson times rounded down to a
    quantum, plus `bursts` runs of `burst_len` equal times (groups > B)"""
    a = np.floor(np.cumsum(rng.exponential(1.0 / rate, n)) / quantum) * quantum
    for _ in range(bursts):
        i = int(rng.integers(0, max(1, n - burst_len)))
        a[i:i + burst_len] = a[i]
    return np.maximum.accumulate(a)


@pytest.mark.parametrize("seed", range(24))
def test_oracle_equals_reference_on_tie_groups(seed):
    """Given arrival arrays with tie groups of any size (App. A.2): the C
    restatement against the reference's own event loop (bbref_run_arrays)."""
    rng = np.random.default_rng(1000 + seed)
    r = random.Random(seed)
    k = r.choice([1, 2, 3, 4, 8])
    B = r.choice([1, 2, 3, 4, 8, 16])
    n = r.randint(max(B, 50), 4000)
    a = tied_arrivals(rng, n, r.uniform(0.5, 4.0), r.choice([0.25, 1.0, 4.0, 16.0]),
                      bursts=r.randint(0, 3), burst_len=r.randint(B + 1, 6 * B + 2))
    if r.random() < 0.2:
        a[-r.randint(B + 1, 5 * B + 1):] = a[-1]  # a final group larger than B
    s = rng.uniform(1.0, 20.0, n)
    cfg = dict(arrival_rate=2.0, n_requests=n, batch_size=B, seed=r.getrandbits(64),
               edges=O.uniform_boundaries(k, 1.0, 20.0).tolist(), service="arrays",
               flush_partial=r.random() < 0.6, n_servers=r.choice([1, 1, 2, 5]))
    if r.random() < 0.5:
        cfg.update(error="symmetric", p_error=r.choice([0.1, 0.4]))
    draws = cfg.get("error") == "symmetric" and k > 1
    u = O.stream_uniform01(O.oracle(), cfg["seed"], 2, n) if draws else None
    mr, dr = O.run(O.reference(), cfg, dict(arrivals=a, services=s))
    mo, do = O.run(O.oracle(), cfg, dict(arrivals=a, services=s, u_err=u))
    for key in REQ_KEYS + BAT_KEYS:
        assert same_bits(do[key], dr[key]), key
    for key in ("makespan", "throughput", "latency_mean", "latency_p50", "latency_p99",
                "server_busy_fraction", "n_completed"):
        assert same_bits(mo[key], mr[key]), key
