"""CPU-side checks of the product library: it loads, exports every symbol
include/binbatch_b200.h declares, its host formulas match the reference, the
Philox KATs hold, and validation raises the reference's exception categories
before any device work.  No compute calls (there is no GPU here)."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

import paper_2412_04504_b200 as bb
from paper_2412_04504_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "binbatch_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_capi.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(_capi.EXPORTS) == names


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _capi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_philox_known_answers():
    # SURVEY App. C (Random123 / curand_philox4x32_x.h KATs)
    assert bb.philox4x32_10([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert bb.philox4x32_10([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2) == [0x408F276D, 0x41C83B0E,
                                                                    0xA20BC7C6, 0x6D5451FD]
    assert bb.philox4x32_10([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344],
                            [0xA4093822, 0x299F31D0]) == [0xD16CFE09, 0x94FDCCEB, 0x5001E420,
                                                          0x24126EA1]


def test_replication_seed_matches_oracle():
    import oracle_py as O
    for m, r in ((1, 0), (1001, 9), (2**64 - 1, 2**40)):
        assert bb.replication_seed(m, r) == O.oracle().replication_seed(m, r)


def test_boundaries_match_reference():
    import oracle_py as O
    if not O.have_reference():
        pytest.skip("reference shim not built")
    ref = O.reference()
    dp = C.POINTER(C.c_double)
    for k, lo, hi in ((1, 1.0, 20.0), (7, 1.0, 20.0), (16, 0.0, 3.3), (5, 0.53, 31.22)):
        out = np.empty(k + 1)
        assert ref.bbref_uniform_boundaries(k, lo, hi, out.ctypes.data_as(dp)) == 0
        assert np.array_equal(np.array(bb.uniform_boundaries(k, lo, hi).edges), out)
    for k, rate, B in ((1, 1.0, 8), (3, 0.1, 200), (8, 2.5, 64)):
        out = np.empty(k + 1)
        assert ref.bbref_exponential_boundaries(k, rate, B, out.ctypes.data_as(dp)) == 0
        assert np.array_equal(np.array(bb.exponential_boundaries(k, rate, B).edges), out)
    rng = np.random.default_rng(3)
    s = rng.pareto(1.2, 5000) + 1.0
    for k in (1, 2, 4, 8, 16, 32):
        out = np.empty(k + 1)
        assert ref.bbref_empirical_boundaries(k, s.ctypes.data_as(dp), len(s), out.ctypes.data_as(dp)) == 0
        assert np.array_equal(np.array(bb.empirical_boundaries(k, s).edges), out)


def test_analytics_kats():
    # test_analytics.cpp:11-84
    assert bb.throughput(128, 1, 1.0, 20.0) == pytest.approx(6.447481452557596, rel=1e-12)
    assert bb.throughput(128, 5, 1.0, 20.0) == pytest.approx(10.347161298408322, rel=1e-12)
    assert bb.expected_latency(128, 1, 1.0, 20.0, 10.0) == pytest.approx(26.202713178294573, rel=1e-12)
    assert bb.expected_latency(128, 2, 1.0, 20.0, 10.0) == pytest.approx(27.876356589147285, rel=1e-12)


def cfg(**kw):
    base = dict(arrival_rate=bb.kOverload, n_requests=100, batch_size=8,
                bins=bb.uniform_boundaries(2, 1.0, 20.0), service=bb.Uniform(1.0, 20.0), seed=1)
    base.update(kw)
    return bb.SimConfig(**base)


@pytest.mark.parametrize("bad", [
    dict(bins=bb.BinConfig([])),                       # no bins
    dict(n_requests=4),                               # n < B
    dict(n_servers=0),
    dict(arrival_rate=0.0),
    dict(max_batch_wait=0.0),
    dict(bins=bb.BinConfig([1.0, 1.0])),              # not strictly increasing
    dict(service=bb.Uniform(5.0, 1.0)),
    dict(error_model=bb.Symmetric(0.7)),
    dict(error_model=bb.Confusion([[0.9, 0.1], [0.2, 0.7]])),
])
def test_validation_categories_match_reference(bad):
    # test_simulator.cpp:31-50 -- invalid_argument before any device work
    with pytest.raises(bb.InvalidArgument):
        bb.run_simulation(cfg(**bad))


def test_replay_trace_validation():
    # test_simulator.cpp:272-274
    c = cfg(n_requests=4, batch_size=2, bins=bb.make_bin_config([1.0, 3.5, 6.0]))
    with pytest.raises(bb.InvalidArgument):
        bb.replay_trace(c, [])
    with pytest.raises(bb.InvalidArgument):
        bb.replay_trace(c, [1.0, -2.0])


def test_outside_gpu_envelope_is_reported():
    # single runs support up to 32 bins (host-side check, before any device work)
    with pytest.raises(NotImplementedError):
        bb.run_simulation(cfg(bins=bb.uniform_boundaries(33, 1.0, 20.0)))


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", None) is None and False, reason="")
def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(bb.CudaError):
        bb.run_simulation(cfg())
    with pytest.raises(bb.CudaError):
        bb.run_experiment(bb.ExperimentSpec(base=bb.RunTemplate(n_requests=64, batch_size=8,
                                                                service=bb.ServiceSpec("uniform", 1.0, 20.0)),
                                            replications=2))


def test_experiment_expansion_and_spec_validation():
    # experiment.hpp:241-252, :316-340 ; test_experiment.cpp:38-55
    base = bb.RunTemplate(n_requests=1280, batch_size=16, flush_partial=False,
                          service=bb.ServiceSpec("uniform", 1.0, 20.0))
    spec = bb.ExperimentSpec(base=base, axes=[bb.SweepAxis("k", [2.0, 1.0])], replications=3, seed=7)
    assert bb.experiment_points(spec) == 2
    spec2 = bb.ExperimentSpec(base=base, axes=[bb.SweepAxis("k", [1, 2, 4, 8, 16]),
                                               bb.SweepAxis("B", [8, 16, 32])], replications=1)
    assert bb.experiment_points(spec2) == 15
    for axes in ([bb.SweepAxis("k", [1.5])], [bb.SweepAxis("lambda", [-1.0])],
                 [bb.SweepAxis("k", [])]):
        with pytest.raises(bb.InvalidArgument):
            bb.experiment_points(bb.ExperimentSpec(base=base, axes=axes))
    with pytest.raises(bb.InvalidArgument):
        bb.experiment_points(bb.ExperimentSpec(base=base, axes=[bb.SweepAxis("k", [1])] * 3))
    with pytest.raises(bb.InvalidArgument):
        bb.experiment_points(bb.ExperimentSpec(base=base, replications=0))
    with pytest.raises(bb.InvalidArgument):
        bb.experiment_points(bb.ExperimentSpec(base=bb.RunTemplate(
            n_requests=10, bins=bb.BinRule(edges=[1.0, 10.0, 20.0])), axes=[bb.SweepAxis("k", [2])]))
