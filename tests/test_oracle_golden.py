"""The C restatement (oracle/bb_oracle.c) reproduces the reference's own
outputs bit-for-bit on the committed golden fixtures (tests/golden/,
generated from /root/reference by tests/golden/make_golden.py)."""
import numpy as np
import pytest

import oracle_py as O
from _helpers import BAT_KEYS, REQ_KEYS, fixture_names, load_fixture, same_bits


@pytest.mark.parametrize("name", fixture_names())
def test_oracle_regenerates_reference_streams_and_results(name):
    cfg, metrics, g = load_fixture(name)
    m, d = O.run(O.oracle(), cfg)
    assert same_bits(d["req_arrival"], g["arrivals"])
    assert same_bits(d["req_service"], g["services"])
    for k in REQ_KEYS + BAT_KEYS:
        assert same_bits(d[k], g[k]), k
    assert same_bits(d["members"], g["members"])
    for k in ("throughput", "makespan", "latency_mean", "latency_p50", "latency_p99",
              "server_busy_fraction", "n_completed", "n_batches"):
        assert same_bits(m[k], metrics[k]), k
    if len(g["u_err"]):
        assert same_bits(O.stream_uniform01(O.oracle(), cfg["seed"], 2, cfg["n_requests"]),
                         g["u_err"])


@pytest.mark.parametrize("name", fixture_names())
def test_oracle_trace_mode_on_golden_streams(name):
    """Trace mode: the same engine driven by the reference's arrays."""
    cfg, metrics, g = load_fixture(name)
    inputs = dict(arrivals=g["arrivals"], services=g["services"],
                  u_err=g["u_err"] if len(g["u_err"]) else None)
    c = dict(cfg, service="arrays")
    m, d = O.run(O.oracle(), c, inputs)
    for k in REQ_KEYS + BAT_KEYS:
        assert same_bits(d[k], g[k]), k
    assert same_bits(m["makespan"], metrics["makespan"])
    assert same_bits(m["latency_mean"], metrics["latency_mean"])
    assert same_bits(m["latency_p99"], metrics["latency_p99"])
