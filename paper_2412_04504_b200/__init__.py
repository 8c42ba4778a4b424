"""B200-native Multi-Bin Batching Monte Carlo engine (arXiv 2412.04504).

Python view of the engine's C ABI (include/binbatch_b200.h), mirroring the
reference simulator's C++ API (/root/reference/proj/include/binbatch/):

    simulator.hpp   SimConfig, SimMetrics, SimResult, run_simulation[_detailed],
                    replay_trace[_detailed], kOverload
    experiment.hpp  RunTemplate, ServiceSpec, BinRule, ErrorSpec, SweepAxis,
                    ExperimentSpec, PointResult, replication_seed, run_point,
                    run_experiment
    binning.hpp     make_bin_config, uniform_/exponential_/empirical_boundaries,
                    Perfect, Symmetric (make_symmetric), Confusion
    analytics.hpp   throughput, expected_latency

Exceptions follow the reference's categories: InvalidArgument
(std::invalid_argument), DomainError (std::domain_error), RuntimeFailure
(std::runtime_error); configurations outside the GPU envelope raise
NotImplementedError.  Every simulation runs in the sm_100a kernels of
libbinbatch_b200.so; without a CUDA device calls raise CudaError.

Request/batch detail is returned structure-of-arrays (numpy), the GPU-native
layout of the reference's Request / BatchRecord vectors.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Union

import numpy as np

from . import _capi

_lib = _capi.load()

kOverload = math.inf
kNoBatch = _capi.BB_NO_BATCH


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class DomainError(ValueError):
    """std::domain_error"""


class RuntimeFailure(RuntimeError):
    """std::runtime_error"""


class CudaError(RuntimeError):
    """no device / CUDA failure"""


def _check(st: int):
    if st == _capi.BB_OK:
        return
    msg = _lib.bb_last_error().decode()
    raise {
        _capi.BB_EINVAL: InvalidArgument,
        _capi.BB_EDOMAIN: DomainError,
        _capi.BB_ERUNTIME: RuntimeFailure,
        _capi.BB_ECUDA: CudaError,
        _capi.BB_EUNSUPPORTED: NotImplementedError,
    }.get(st, RuntimeFailure)(msg)


def _dptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


# --------------------------------------------------------------- binning
@dataclass
class BinConfig:
    """binning.hpp:23-29"""
    edges: List[float]

    def bin_count(self) -> int:
        return len(self.edges) - 1


def make_bin_config(edges: Sequence[float]) -> BinConfig:
    """binning.hpp:31-44 (validated by the library on use, and here)"""
    e = [float(x) for x in edges]
    if len(e) < 2:
        raise InvalidArgument("bin config: need at least two edges")
    for i, v in enumerate(e):
        last = i + 1 == len(e)
        if math.isnan(v) or (not last and not math.isfinite(v)) or (last and v == -math.inf):
            raise InvalidArgument("bin config: only the top edge may be infinite")
    for i in range(1, len(e)):
        if not e[i - 1] < e[i]:
            raise InvalidArgument("bin config: edges must be strictly increasing")
    return BinConfig(e)


def _edges_call(fn, k, *args):
    out = np.empty(int(k) + 1)
    _check(fn(int(k), *args, out.ctypes.data_as(C.POINTER(C.c_double))))
    return BinConfig(out.tolist())


def uniform_boundaries(k: int, min_time: float, max_time: float) -> BinConfig:
    """binning.hpp:47-57"""
    if k < 1:
        raise InvalidArgument("uniform_boundaries: k must be >= 1")
    return _edges_call(_lib.bb_uniform_boundaries, k, float(min_time), float(max_time))


def exponential_boundaries(k: int, rate: float, batch_size: int) -> BinConfig:
    """binning.hpp:79-93"""
    if k < 1:
        raise InvalidArgument("exponential_boundaries: k must be >= 1")
    return _edges_call(_lib.bb_exponential_boundaries, k, float(rate), int(batch_size))


def empirical_boundaries(k: int, samples: Sequence[float]) -> BinConfig:
    """binning.hpp:110-128"""
    if k < 1:
        raise InvalidArgument("empirical_boundaries: k must be >= 1")
    s = np.ascontiguousarray(samples, dtype=np.float64)
    return _edges_call(_lib.bb_empirical_boundaries, k, _dptr(s), len(s))


@dataclass
class Perfect:
    pass


@dataclass
class Symmetric:
    p_error: float = 0.0


@dataclass
class Confusion:
    rows: List[List[float]]


ErrorModel = Union[Perfect, Symmetric, Confusion]


def make_symmetric(p_error: float) -> Symmetric:
    """binning.hpp:164-168"""
    if not (p_error >= 0 and p_error <= 0.5):
        raise InvalidArgument("symmetric error model: need 0 <= p_error <= 0.5")
    return Symmetric(float(p_error))


def make_confusion(rows) -> Confusion:
    """binning.hpp:170-188"""
    rows = [list(map(float, r)) for r in rows]
    if not rows:
        raise InvalidArgument("confusion matrix: empty")
    k = len(rows)
    for i, r in enumerate(rows):
        if len(r) != k:
            raise InvalidArgument("confusion matrix: must be square")
        if any(not (p >= 0) for p in r):
            raise InvalidArgument("confusion matrix: negative entry")
        if abs(sum(r) - 1.0) > 1e-9:
            raise InvalidArgument(f"confusion matrix: row {i + 1} sums to {sum(r)}, expected 1")
    return Confusion(rows)


# ---------------------------------------------------------- service models
@dataclass
class Uniform:
    min_time: float = 1.0
    max_time: float = 2.0


@dataclass
class Exponential:
    rate: float = 1.0


@dataclass
class Empirical:
    samples: List[float] = field(default_factory=list)


@dataclass
class Linear:
    """t = slope*len + intercept with len ~ U[min_len, max_len] (tokens_to_time, workload.hpp:167)"""
    min_len: float = 1.0
    max_len: float = 1024.0
    intercept: float = 0.5
    slope: float = 0.03


@dataclass
class LogNormal:
    mu: float = 0.0
    sigma: float = 1.0


ServiceDist = Union[Uniform, Exponential, Empirical, Linear, LogNormal]


def make_uniform(min_time, max_time) -> Uniform:
    if not (min_time >= 0 and min_time < max_time and math.isfinite(max_time)):
        raise InvalidArgument("uniform service: need 0 <= min_time < max_time")
    return Uniform(float(min_time), float(max_time))


def make_exponential(rate) -> Exponential:
    if not (rate > 0 and math.isfinite(rate)):
        raise InvalidArgument("exponential service: rate must be positive")
    return Exponential(float(rate))


def make_empirical(samples) -> Empirical:
    s = [float(x) for x in samples]
    if not s:
        raise InvalidArgument("empirical service: sample set is empty")
    if any(not (x > 0 and math.isfinite(x)) for x in s):
        raise InvalidArgument("empirical service: all samples must be positive")
    return Empirical(sorted(s))


# -------------------------------------------------------------- simulator
@dataclass
class SimConfig:
    """simulator.hpp:62-74 (+ rng / device, see include/binbatch_b200.h)"""
    arrival_rate: float = kOverload
    n_requests: int = 0
    batch_size: int = 1
    bins: BinConfig = field(default_factory=lambda: BinConfig([]))
    error_model: ErrorModel = field(default_factory=Perfect)
    n_servers: int = 1
    service: ServiceDist = field(default_factory=lambda: Uniform(1.0, 2.0))
    seed: int = 0
    flush_partial: bool = True
    max_batch_wait: Optional[float] = None
    trace_mode: str = "cyclic"
    rng: str = "philox"
    device: int = -1


@dataclass
class SimMetrics:
    """simulator.hpp:76-87"""
    throughput: float = 0.0
    makespan: float = 0.0
    latency_mean: float = 0.0
    latency_p50: float = 0.0
    latency_p99: float = 0.0
    per_bin_batch_counts: List[int] = field(default_factory=list)
    server_busy_fraction: float = 0.0
    n_completed: int = 0


@dataclass
class SimResult:
    """simulator.hpp:89-93 -- requests/batches as structure-of-arrays"""
    metrics: SimMetrics
    requests: dict
    batches: dict


class _Keep:
    pass


def _cfg_struct(cfg: SimConfig, table=None):
    keep = _Keep()
    c = _capi.SimConfigC()
    c.arrival_rate = float(cfg.arrival_rate)
    c.n_requests = int(cfg.n_requests)
    c.batch_size = int(cfg.batch_size)
    c.n_servers = int(cfg.n_servers)
    c.seed = int(cfg.seed) & (2**64 - 1)
    c.flush_partial = int(bool(cfg.flush_partial))
    c.has_max_batch_wait = int(cfg.max_batch_wait is not None)
    c.max_batch_wait = float(cfg.max_batch_wait or 0.0)
    keep.edges = np.ascontiguousarray(cfg.bins.edges, dtype=np.float64)
    c.edges = _dptr(keep.edges) if len(keep.edges) else None
    c.n_edges = len(keep.edges)
    em = cfg.error_model
    if isinstance(em, Symmetric):
        c.error_kind, c.p_error = 1, float(em.p_error)
    elif isinstance(em, Confusion):
        c.error_kind = 2
        keep.conf = np.ascontiguousarray(em.rows, dtype=np.float64).ravel()
        c.confusion = _dptr(keep.conf)
        c.confusion_k = len(em.rows)
    else:
        c.error_kind = 0
    sv = cfg.service
    if isinstance(sv, Uniform):
        c.service_kind, c.lo, c.hi = 0, float(sv.min_time), float(sv.max_time)
    elif isinstance(sv, Exponential):
        c.service_kind, c.rate = 1, float(sv.rate)
    elif isinstance(sv, Empirical):
        c.service_kind = 2
        table = sv.samples
    elif isinstance(sv, Linear):
        c.service_kind, c.lo, c.hi = 6, float(sv.min_len), float(sv.max_len)
        c.lin_a, c.lin_b = float(sv.intercept), float(sv.slope)
    elif isinstance(sv, LogNormal):
        c.service_kind, c.mu, c.sigma = 7, float(sv.mu), float(sv.sigma)
    if table is not None:
        keep.table = np.ascontiguousarray(table, dtype=np.float64)
        c.table = _dptr(keep.table)
        c.n_table = len(keep.table)
    c.rng = _capi.RNG[cfg.rng]
    c.device = int(cfg.device)
    return c, keep


def _metrics(m: _capi.SimMetricsC) -> SimMetrics:
    return SimMetrics(
        throughput=m.throughput, makespan=m.makespan, latency_mean=m.latency_mean,
        latency_p50=m.latency_p50, latency_p99=m.latency_p99,
        per_bin_batch_counts=[int(m.per_bin_batch_counts[i]) for i in range(m.k)],
        server_busy_fraction=m.server_busy_fraction, n_completed=int(m.n_completed))


def _detail(n: int):
    d = dict(
        arrival=np.empty(n), service=np.empty(n), true_bin=np.empty(n, np.uint8),
        predicted_bin=np.empty(n, np.uint8), batch=np.empty(n, np.uint32),
        completion=np.empty(n), b_bin=np.empty(n, np.uint8), b_size=np.empty(n, np.uint32),
        b_first=np.empty(n, np.uint32), b_formed=np.empty(n), b_start=np.empty(n),
        b_finish=np.empty(n), b_service=np.empty(n), members=np.empty(n, np.uint32))
    D = _capi.SimDetailC()
    P = C.POINTER
    D.req_arrival = _dptr(d["arrival"])
    D.req_service = _dptr(d["service"])
    D.req_true_bin = d["true_bin"].ctypes.data_as(P(C.c_uint8))
    D.req_pred_bin = d["predicted_bin"].ctypes.data_as(P(C.c_uint8))
    D.req_batch = d["batch"].ctypes.data_as(P(C.c_uint32))
    D.req_completion = _dptr(d["completion"])
    D.batch_capacity = n
    D.bat_bin = d["b_bin"].ctypes.data_as(P(C.c_uint8))
    D.bat_size = d["b_size"].ctypes.data_as(P(C.c_uint32))
    D.bat_first = d["b_first"].ctypes.data_as(P(C.c_uint32))
    D.bat_formed = _dptr(d["b_formed"])
    D.bat_start = _dptr(d["b_start"])
    D.bat_finish = _dptr(d["b_finish"])
    D.bat_service = _dptr(d["b_service"])
    D.members = d["members"].ctypes.data_as(P(C.c_uint32))
    return d, D


def _result(m, d) -> SimResult:
    nb = int(m.n_batches)
    requests = {k: d[k] for k in ("arrival", "service", "true_bin", "predicted_bin", "batch",
                                  "completion")}
    batches = {"bin": d["b_bin"][:nb], "size": d["b_size"][:nb], "first": d["b_first"][:nb],
               "formed_time": d["b_formed"][:nb], "start_time": d["b_start"][:nb],
               "finish_time": d["b_finish"][:nb], "service_time": d["b_service"][:nb],
               "members": d["members"][: int(d["b_size"][:nb].sum())]}
    return SimResult(_metrics(m), requests, batches)


def run_simulation(cfg: SimConfig) -> SimMetrics:
    """simulator.hpp:338"""
    c, keep = _cfg_struct(cfg)
    m = _capi.SimMetricsC()
    _check(_lib.bb_run_simulation(C.byref(c), C.byref(m)))
    return _metrics(m)


def run_simulation_detailed(cfg: SimConfig) -> SimResult:
    """simulator.hpp:331"""
    c, keep = _cfg_struct(cfg)
    m = _capi.SimMetricsC()
    d, D = _detail(int(cfg.n_requests))
    _check(_lib.bb_run_simulation_detailed(C.byref(c), C.byref(m), C.byref(D)))
    return _result(m, d)


def _trace_cfg(cfg: SimConfig, lengths):
    c, keep = _cfg_struct(cfg, table=lengths)
    c.service_kind = _capi.SVC["trace_resample" if cfg.trace_mode == "resample" else "trace_cyclic"]
    return c, keep


def replay_trace(cfg: SimConfig, lengths: Sequence[float]) -> SimMetrics:
    """simulator.hpp:356"""
    lengths = np.ascontiguousarray(lengths, dtype=np.float64)
    c, keep = _trace_cfg(cfg, lengths)
    m = _capi.SimMetricsC()
    _check(_lib.bb_replay_trace(C.byref(c), _dptr(lengths) if len(lengths) else None,
                                len(lengths), C.byref(m)))
    return _metrics(m)


def replay_trace_detailed(cfg: SimConfig, lengths: Sequence[float]) -> SimResult:
    """simulator.hpp:344"""
    lengths = np.ascontiguousarray(lengths, dtype=np.float64)
    c, keep = _trace_cfg(cfg, lengths)
    m = _capi.SimMetricsC()
    d, D = _detail(int(cfg.n_requests))
    _check(_lib.bb_replay_trace_detailed(C.byref(c), _dptr(lengths) if len(lengths) else None,
                                         len(lengths), C.byref(m), C.byref(D)))
    return _result(m, d)


def run_trace(cfg: SimConfig, arrivals, services, u_err=None, pred_bin=None,
              detailed: bool = False):
    """Engine::run (simulator.hpp:128) on given request streams -- trace mode."""
    a = np.ascontiguousarray(arrivals, dtype=np.float64)
    s = np.ascontiguousarray(services, dtype=np.float64)
    u = None if u_err is None else np.ascontiguousarray(u_err, dtype=np.float64)
    p = None if pred_bin is None else np.ascontiguousarray(pred_bin, dtype=np.uint8)
    c, keep = _cfg_struct(cfg)
    tin = _capi.TraceInC(_dptr(a), _dptr(s), _dptr(u),
                         None if p is None else p.ctypes.data_as(C.POINTER(C.c_uint8)))
    m = _capi.SimMetricsC()
    if detailed:
        d, D = _detail(int(cfg.n_requests))
        _check(_lib.bb_run_trace(C.byref(c), C.byref(tin), C.byref(m), C.byref(D)))
        return _result(m, d)
    _check(_lib.bb_run_trace(C.byref(c), C.byref(tin), C.byref(m), None))
    return _metrics(m)


def run_trace_device(cfg: SimConfig, arrivals_ptr: int, services_ptr: int, u_err_ptr: int = 0,
                     pred_ptr: int = 0, stream: int = 0) -> SimMetrics:
    """Trace mode on device-resident arrays (raw CUDA pointers), stream-ordered."""
    c, keep = _cfg_struct(cfg)
    dp = C.POINTER(C.c_double)
    tin = _capi.TraceInC(C.cast(arrivals_ptr, dp), C.cast(services_ptr, dp),
                         C.cast(u_err_ptr, dp) if u_err_ptr else None,
                         C.cast(pred_ptr, C.POINTER(C.c_uint8)) if pred_ptr else None)
    m = _capi.SimMetricsC()
    _check(_lib.bb_run_trace_device(C.byref(c), C.byref(tin), C.byref(m), None,
                                    C.c_void_p(stream) if stream else None))
    return _metrics(m)


# -------------------------------------------------------------- experiments
@dataclass
class ServiceSpec:
    """experiment.hpp:36-45 (+ linear / lognormal kinds)"""
    kind: str = "uniform"          # uniform | exponential | trace | linear | lognormal
    min_time: float = 1.0
    max_time: float = 2.0
    rate: float = 1.0
    trace_times: Optional[List[float]] = None
    trace_mode: str = "resample"   # ServiceSpec default (experiment.hpp:43)
    intercept: float = 0.5
    slope: float = 0.03
    mu: float = 0.0
    sigma: float = 1.0


@dataclass
class BinRule:
    k: int = 1
    edges: List[float] = field(default_factory=list)


@dataclass
class ErrorSpec:
    kind: str = "perfect"
    p_error: float = 0.0
    rows: Optional[List[List[float]]] = None


@dataclass
class RunTemplate:
    """experiment.hpp:63-73"""
    arrival_rate: float = kOverload
    n_requests: int = 0
    batch_size: int = 1
    n_servers: int = 1
    flush_partial: bool = True
    max_batch_wait: Optional[float] = None
    service: ServiceSpec = field(default_factory=ServiceSpec)
    bins: BinRule = field(default_factory=BinRule)
    error: ErrorSpec = field(default_factory=ErrorSpec)


@dataclass
class SweepAxis:
    param: str
    values: List[float]


@dataclass
class ExperimentSpec:
    """experiment.hpp:80-87"""
    name: str = "experiment"
    base: RunTemplate = field(default_factory=RunTemplate)
    axes: List[SweepAxis] = field(default_factory=list)
    replications: int = 10
    output: str = ""
    seed: int = 1
    rng: str = "philox"


@dataclass
class PointResult:
    """experiment.hpp:166-184"""
    arrival_rate: float
    k: int
    batch_size: int
    n_servers: int
    error_model: str
    p_error: float
    n_requests: int
    replications: int
    throughput_mean: float
    throughput_std: float
    latency_mean: float
    latency_std: float
    latency_p50: float
    latency_p99: float
    makespan_mean: float
    busy_fraction_mean: float
    analytic_throughput: float
    analytic_latency: float
    analytic_max_throughput: float


def _template_struct(t: RunTemplate, keep: _Keep) -> _capi.RunTemplateC:
    c = _capi.RunTemplateC()
    c.arrival_rate = float(t.arrival_rate)
    c.n_requests = int(t.n_requests)
    c.batch_size = int(t.batch_size)
    c.n_servers = int(t.n_servers)
    c.flush_partial = int(bool(t.flush_partial))
    c.has_max_batch_wait = int(t.max_batch_wait is not None)
    c.max_batch_wait = float(t.max_batch_wait or 0.0)
    s = t.service
    c.service = _capi.KIND[s.kind]
    c.trace_cyclic = int(s.trace_mode == "cyclic")
    c.min_time, c.max_time, c.rate = float(s.min_time), float(s.max_time), float(s.rate)
    c.lin_a, c.lin_b, c.mu, c.sigma = float(s.intercept), float(s.slope), float(s.mu), float(s.sigma)
    if s.trace_times is not None:
        keep.trace = np.ascontiguousarray(s.trace_times, dtype=np.float64)
        c.trace_times = _dptr(keep.trace)
        c.n_trace = len(keep.trace)
    c.k = int(t.bins.k)
    if t.bins.edges:
        keep.edges = np.ascontiguousarray(t.bins.edges, dtype=np.float64)
        c.edges = _dptr(keep.edges)
        c.n_edges = len(keep.edges)
    c.error_kind = _capi.ERR[t.error.kind]
    c.p_error = float(t.error.p_error)
    if t.error.rows is not None:
        keep.conf = np.ascontiguousarray(t.error.rows, dtype=np.float64).ravel()
        c.confusion = _dptr(keep.conf)
        c.confusion_k = len(t.error.rows)
    return c


def _spec_struct(spec: ExperimentSpec):
    keep = _Keep()
    E = _capi.ExperimentSpecC()
    E.base = _template_struct(spec.base, keep)
    keep.axes = []
    for i, ax in enumerate(spec.axes[:2]):
        if ax.param not in _capi.AXIS:
            raise InvalidArgument(f"unknown sweep parameter: {ax.param}")
        v = np.ascontiguousarray(ax.values, dtype=np.float64)
        keep.axes.append(v)
        E.axes[i] = _capi.SweepAxisC(_capi.AXIS[ax.param], _dptr(v) if len(v) else None, len(v))
    E.n_axes = len(spec.axes)
    E.replications = int(spec.replications)
    E.seed = int(spec.seed) & (2**64 - 1)
    E.rng = _capi.RNG[spec.rng]
    keep.name = str(spec.name).encode()
    E.name = keep.name
    return E, keep


_ERR_NAMES = {0: "perfect", 1: "symmetric", 2: "confusion"}


def _point(r: _capi.PointResultC) -> PointResult:
    return PointResult(
        r.arrival_rate, int(r.k), int(r.batch_size), int(r.n_servers), _ERR_NAMES[r.error_kind],
        r.p_error, int(r.n_requests), int(r.replications), r.throughput_mean, r.throughput_std,
        r.latency_mean, r.latency_std, r.latency_p50, r.latency_p99, r.makespan_mean,
        r.busy_fraction_mean, r.analytic_throughput, r.analytic_latency,
        r.analytic_max_throughput)


def experiment_points(spec: ExperimentSpec) -> int:
    E, keep = _spec_struct(spec)
    n = C.c_uint64()
    _check(_lib.bb_experiment_points(C.byref(E), C.byref(n)))
    return n.value


def run_experiment(spec: ExperimentSpec, jobs: int = 1) -> List[PointResult]:
    """experiment.hpp:312-370 (one device launch for every point x replication)"""
    E, keep = _spec_struct(spec)
    n = C.c_uint64()
    _check(_lib.bb_run_experiment(C.byref(E), int(jobs), None, 0, C.byref(n)))
    out = (_capi.PointResultC * max(1, n.value))()
    _check(_lib.bb_run_experiment(C.byref(E), int(jobs), out, n.value, C.byref(n)))
    return [_point(out[i]) for i in range(n.value)]


def run_point(t: RunTemplate, master_seed: int, replications: int, rng: str = "philox") -> PointResult:
    """experiment.hpp:254-307 (errors propagate unwrapped, like the reference's run_point)"""
    return run_points([t], replications, master_seed, rng=rng)[0]


def sweep_shard_device(spec: ExperimentSpec, rep_begin: int, rep_end: int, rep_ptr: int,
                       stream: int = 0) -> None:
    """Replications [rep_begin, rep_end) of every point into a device array
    ([6][points*replications] float64 at rep_ptr); stream-ordered."""
    E, keep = _spec_struct(spec)
    _check(_lib.bb_sweep_shard_device(C.byref(E), rep_begin, rep_end, C.c_void_p(rep_ptr),
                                      C.c_void_p(stream) if stream else None))


def sweep_reduce_device(spec: ExperimentSpec, rep_ptr: int, stream: int = 0) -> List[PointResult]:
    E, keep = _spec_struct(spec)
    n = experiment_points(spec)
    out = (_capi.PointResultC * max(1, n))()
    _check(_lib.bb_sweep_reduce_device(C.byref(E), C.c_void_p(rep_ptr), out,
                                       C.c_void_p(stream) if stream else None))
    return [_point(out[i]) for i in range(n)]


def _points_array(points: Sequence[RunTemplate]):
    keep = _Keep()
    keep.items = [_Keep() for _ in points]
    arr = (_capi.RunTemplateC * len(points))()
    for i, t in enumerate(points):
        arr[i] = _template_struct(t, keep.items[i])
    return arr, keep


def run_points(points: Sequence[RunTemplate], replications: int, seed: int,
               rng: str = "philox") -> List[PointResult]:
    """run_point over an explicit list of templates, all in one launch (host results)."""
    arr, keep = _points_array(points)
    out = (_capi.PointResultC * len(points))()
    _check(_lib.bb_run_points(arr, len(points), int(replications), int(seed) & (2**64 - 1),
                              _capi.RNG[rng], out))
    return [_point(out[i]) for i in range(len(points))]


def points_shard_device(points: Sequence[RunTemplate], replications: int, seed: int,
                        rep_begin: int, rep_end: int, rep_ptr: int, stream: int = 0) -> None:
    arr, keep = _points_array(points)
    _check(_lib.bb_points_shard_device(arr, len(points), int(replications),
                                       int(seed) & (2**64 - 1), rep_begin, rep_end,
                                       C.c_void_p(rep_ptr), C.c_void_p(stream) if stream else None))


def points_reduce_device(points: Sequence[RunTemplate], replications: int, rep_ptr: int,
                         stream: int = 0) -> List[PointResult]:
    arr, keep = _points_array(points)
    out = (_capi.PointResultC * len(points))()
    _check(_lib.bb_points_reduce_device(arr, len(points), int(replications), C.c_void_p(rep_ptr),
                                        out, C.c_void_p(stream) if stream else None))
    return [_point(out[i]) for i in range(len(points))]


def points_shard_local_device(points: Sequence[RunTemplate], replications: int, seed: int,
                              rep_begin: int, rep_end: int, shard_ptr: int, stream: int = 0) -> None:
    """Shard [rep_begin, rep_end) into its own block [6][points][rep_end-rep_begin]
    (what an all-gather of the ranks' blocks concatenates)."""
    arr, keep = _points_array(points)
    _check(_lib.bb_points_shard_local_device(arr, len(points), int(replications),
                                             int(seed) & (2**64 - 1), rep_begin, rep_end,
                                             C.c_void_p(shard_ptr), C.c_void_p(stream) if stream else None))


def points_reduce_gathered_device(points: Sequence[RunTemplate], replications: int, n_shards: int,
                                  gathered_ptr: int, stream: int = 0) -> List[PointResult]:
    """run_point's per-point reduction over the concatenated blocks of n_shards
    shards [R c / C, R (c+1) / C) (replication order, bit-identical to one device)."""
    arr, keep = _points_array(points)
    out = (_capi.PointResultC * len(points))()
    _check(_lib.bb_points_reduce_gathered_device(arr, len(points), int(replications), int(n_shards),
                                                 C.c_void_p(gathered_ptr), out,
                                                 C.c_void_p(stream) if stream else None))
    return [_point(out[i]) for i in range(len(points))]


def set_devices(devices: Sequence[int] = ()) -> None:
    """Devices host-side sweeps (run_experiment / run_points / run_point) spread
    their replications over: one host thread per entry, gathered on devices[0].
    Entries may repeat; () restores the current device."""
    arr = (C.c_int32 * max(1, len(devices)))(*[int(d) for d in devices])
    _check(_lib.bb_set_devices(arr, len(devices)))


def replication_seed(master: int, rep: int) -> int:
    """experiment.hpp:90-92"""
    return int(_lib.bb_replication_seed(master & (2**64 - 1), rep & (2**64 - 1)))


# ---------------------------------------------------------------- analytics
def throughput(batch_size: int, bins: int, min_time: float, max_time: float) -> float:
    """analytics.hpp:65-69"""
    return _lib.bb_analytic_throughput(batch_size, bins, min_time, max_time)


def expected_latency(batch_size, bins, min_time, max_time, arrival_rate) -> float:
    """analytics.hpp:101-108"""
    return _lib.bb_analytic_latency(batch_size, bins, min_time, max_time, arrival_rate)


def philox4x32_10(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    _lib.bb_philox4x32_10(c, k, o)
    return list(o)


def exponential_variates(keys, table: bool = True):
    """E = -log1p(-x 2^-53) for 53-bit keys x, computed on the device by the
    engine's gap function (table=True) or its service-key function."""
    import numpy as np
    x = np.ascontiguousarray(keys, dtype=np.uint64)
    out = np.empty(x.shape[0], dtype=np.float64)
    _check(_lib.bb_exponential_variates(x.ctypes.data_as(C.POINTER(C.c_uint64)), x.shape[0],
                                        int(bool(table)),
                                        out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def template_edges(t: RunTemplate) -> List[float]:
    """The edges `t` materialises to (experiment.hpp:128-146)."""
    keep = _Keep()
    c = _template_struct(t, keep)
    n = C.c_uint64()
    _check(_lib.bb_template_edges(C.byref(c), None, 0, C.byref(n)))
    out = np.empty(n.value)
    _check(_lib.bb_template_edges(C.byref(c), _dptr(out), n.value, C.byref(n)))
    return out.tolist()


def service_of_keys(t: RunTemplate, keys) -> np.ndarray:
    """The service time the generated-mode kernels give each 53-bit key."""
    keep = _Keep()
    c = _template_struct(t, keep)
    x = np.ascontiguousarray(keys, dtype=np.uint64)
    out = np.empty(x.shape[0])
    _check(_lib.bb_service_of_keys(C.byref(c), x.ctypes.data_as(C.POINTER(C.c_uint64)),
                                   x.shape[0], _dptr(out)))
    return out


def set_generated_quantiles(on: bool) -> bool:
    """Exact per-replication p50/p99 in generated mode (default on, like the
    reference's finish()); off leaves them NaN (A/B measurement only).
    Returns the previous setting."""
    return bool(_lib.bb_set_generated_quantiles(int(bool(on))))


def launch_count(reset: bool = False) -> int:
    return int(_lib.bb_launch_count(int(reset)))


def transfer_bytes(reset: bool = False):
    h, d = C.c_uint64(), C.c_uint64()
    _lib.bb_transfer_bytes(C.byref(h), C.byref(d), int(reset))
    return h.value, d.value


def trace_graph_stats(reset: bool = False):
    """(captures, replays) of the trace pipeline's CUDA graph (cumulative)."""
    c, r = C.c_uint64(), C.c_uint64()
    _lib.bb_trace_graph_stats(C.byref(c), C.byref(r), int(reset))
    return c.value, r.value


def last_kernel_ms():
    name = C.c_char_p()
    ms = _lib.bb_last_kernel_ms(C.byref(name))
    return ms, (name.value or b"").decode()


def library_path() -> str:
    return _capi.LIB_PATH
