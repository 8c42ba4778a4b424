"""Known-answer tests from the reference's own test suite, against the oracle
(test_simulator.cpp, test_binning.cpp, test_analytics.cpp, acceptance.cpp)."""
import math

import numpy as np
import pytest

import oracle_py as O


def run(cfg):
    return O.run(O.oracle(), cfg)


def test_worked_example_11_vs_8():
    # test_simulator.cpp:313-328, acceptance.cpp:300-320
    base = dict(arrival_rate=math.inf, n_requests=4, batch_size=2, seed=2,
                service="trace_cyclic", table=[1.0, 5.0, 2.0, 6.0])
    assert run(dict(base, edges=[1.0, 6.0]))[0]["makespan"] == 11.0
    assert run(dict(base, edges=[1.0, 3.5, 6.0]))[0]["makespan"] == 8.0


def test_two_length_trace_24_vs_14():
    # test_simulator.cpp:293-311
    base = dict(arrival_rate=math.inf, n_requests=8, batch_size=2, seed=1,
                service="trace_cyclic", table=[1.0, 6.0])
    assert run(dict(base, edges=[1.0, 6.0]))[0]["makespan"] == 24.0
    assert run(dict(base, edges=[1.0, 3.5, 6.0]))[0]["makespan"] == 14.0


def test_equal_length_trace_two_servers():
    # test_simulator.cpp:277-291
    m, d = run(dict(arrival_rate=math.inf, n_requests=64, batch_size=16, edges=[0.5, 1.5],
                    n_servers=2, seed=31, service="trace_cyclic", table=[1.0]))
    assert np.all(d["bat_service"] == 1.0)
    assert m["makespan"] == pytest.approx(2.0)
    assert m["throughput"] == pytest.approx(32.0)


def test_assign_bin_kats():
    # test_binning.cpp:127-139
    e = np.array([1.0, 10.5, 20.0])
    lib = O.oracle()
    import ctypes as C
    b = C.c_uint32()
    for length, want in ((5.0, 1), (10.5, 2), (20.0, 2), (1.0, 1)):
        assert lib.bbo_assign_bin(e.ctypes.data_as(C.POINTER(C.c_double)), 3, C.c_double(length),
                                  C.byref(b)) == 0
        assert b.value == want
    for length in (0.5, 20.5, math.nan):
        assert lib.bbo_assign_bin(e.ctypes.data_as(C.POINTER(C.c_double)), 3, C.c_double(length),
                                  C.byref(b)) == O.EDOMAIN
    op = np.array([0.0, 1.0, math.inf])
    for length, want in ((1e12, 2), (0.0, 1)):
        assert lib.bbo_assign_bin(op.ctypes.data_as(C.POINTER(C.c_double)), 3, C.c_double(length),
                                  C.byref(b)) == 0
        assert b.value == want


def test_validation_errors():
    # test_simulator.cpp:31-50
    ok = dict(arrival_rate=math.inf, n_requests=100, batch_size=8, edges=[1.0, 10.5, 20.0],
              lo=1.0, hi=20.0, seed=1)
    for bad in (dict(n_requests=4), dict(n_servers=0), dict(arrival_rate=0.0),
                dict(max_batch_wait=0.0), dict(edges=[1.0])):
        with pytest.raises(O.OracleError) as ei:
            run(dict(ok, **bad))
        assert ei.value.code == O.EINVAL
    run(dict(ok, error="confusion", confusion=[[0.9, 0.1], [0.1, 0.9]]))


def test_out_of_support_is_domain_error():
    # test_simulator.cpp:265-275
    cfg = dict(arrival_rate=math.inf, n_requests=4, batch_size=2, edges=[1.0, 3.5, 6.0], seed=5,
               service="trace_cyclic", table=[1.0, 5.0, 2.0, 50.0])
    with pytest.raises(O.OracleError) as ei:
        run(cfg)
    assert ei.value.code == O.EDOMAIN
    with pytest.raises(O.OracleError) as ei:
        run(dict(cfg, table=[1.0, -2.0]))
    assert ei.value.code == O.EINVAL


def test_overload_makespan_is_total_service():
    # test_simulator.cpp:177-184
    m, d = run(dict(arrival_rate=math.inf, n_requests=5 * 128, batch_size=128,
                    edges=O.uniform_boundaries(2, 1, 20), lo=1.0, hi=20.0, seed=77))
    assert m["makespan"] == pytest.approx(d["bat_service"].sum(), rel=1e-12)
    assert m["server_busy_fraction"] == pytest.approx(1.0, rel=1e-12)


def test_no_flush_leaves_only_full_batches():
    # test_simulator.cpp:231-242
    m, d = run(dict(arrival_rate=math.inf, n_requests=1000, batch_size=16,
                    edges=O.uniform_boundaries(3, 1, 20), lo=1.0, hi=20.0, seed=9,
                    flush_partial=False))
    assert np.all(d["bat_size"] == 16)
    assert m["n_completed"] == 16 * m["n_batches"] < 1000
    assert np.sum(d["req_batch"] == np.uint64(2**64 - 1)) == 1000 - m["n_completed"]


def test_replication_seed_and_streams_match_reference():
    o = O.oracle()
    if not O.have_reference():
        pytest.skip("reference shim not built")
    r = O.reference()
    for m, k in ((1, 0), (1001, 7), (2**63 + 5, 123456)):
        assert o.replication_seed(m, k) == r.replication_seed(m, k)
    for seed in (0, 1001, 2**64 - 1):
        for stream in (0, 1, 2):
            assert np.array_equal(O.stream_uniform01(o, seed, stream, 1000),
                                  O.stream_uniform01(r, seed, stream, 1000))
