"""TEST INFRASTRUCTURE ONLY -- ctypes view of the CPU oracle libraries.

* ``oracle/_build/liboracle.so`` -- the plain-C restatement (bb_oracle.c).
* ``oracle/_ref/libbbref.so``   -- the unmodified reference headers behind a
  thin extern "C" shim (ref_shim.cpp), compiled in place from
  /root/reference by oracle/Makefile.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module, and only as the checker or the
CPU baseline -- never as the thing measured or shipped.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbbref.so")

OK, EINVAL, EDOMAIN, ERUNTIME, EUNSUPPORTED = 0, 1, 2, 3, 4
SVC = dict(uniform=0, exponential=1, empirical=2, trace_cyclic=3, trace_resample=4,
           arrays=5, linear=6, lognormal=7)
ERR = dict(perfect=0, symmetric=1, confusion=2)

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_u8p = C.POINTER(C.c_uint8)


class Cfg(C.Structure):
    _fields_ = [
        ("arrival_rate", C.c_double), ("n_requests", C.c_uint64), ("batch_size", C.c_uint64),
        ("n_servers", C.c_uint64), ("seed", C.c_uint64), ("flush_partial", C.c_int32),
        ("has_max_batch_wait", C.c_int32), ("max_batch_wait", C.c_double),
        ("edges", _dp), ("n_edges", C.c_uint64), ("error_kind", C.c_int32),
        ("service_kind", C.c_int32), ("p_error", C.c_double), ("confusion", _dp),
        ("lo", C.c_double), ("hi", C.c_double), ("rate", C.c_double),
        ("lin_a", C.c_double), ("lin_b", C.c_double), ("mu", C.c_double), ("sigma", C.c_double),
        ("table", _dp), ("n_table", C.c_uint64),
    ]


class Inputs(C.Structure):
    _fields_ = [("arrivals", _dp), ("services", _dp), ("u_err", _dp), ("pred_bin", _u8p)]


class Metrics(C.Structure):
    _fields_ = [
        ("throughput", C.c_double), ("makespan", C.c_double), ("latency_mean", C.c_double),
        ("latency_p50", C.c_double), ("latency_p99", C.c_double),
        ("server_busy_fraction", C.c_double), ("n_completed", C.c_uint64),
        ("n_batches", C.c_uint64), ("busy_time", C.c_double), ("latency_sum", C.c_double),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Detail(C.Structure):
    _fields_ = [
        ("req_arrival", _dp), ("req_service", _dp), ("req_true_bin", _u32p),
        ("req_pred_bin", _u32p), ("req_batch", _u64p), ("req_completion", _dp),
        ("bat_bin", _u32p), ("bat_size", _u64p), ("bat_first", _u64p), ("bat_formed", _dp),
        ("bat_start", _dp), ("bat_finish", _dp), ("bat_service", _dp), ("members", _u64p),
        ("per_bin_batch_counts", _u64p),
    ]


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def _load(path, prefix):
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing -- run `make -C oracle`")
    lib = C.CDLL(path)
    run = getattr(lib, prefix + "run")
    last = getattr(lib, prefix + "last_error")
    last.restype = C.c_char_p
    lib.replication_seed = getattr(lib, prefix + "replication_seed")
    lib.replication_seed.restype = C.c_uint64
    lib.replication_seed.argtypes = [C.c_uint64, C.c_uint64]
    lib.stream_uniform01 = getattr(lib, prefix + "stream_uniform01")
    lib.stream_uniform01.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _dp]
    lib.last = last
    lib.prefix = prefix
    if prefix == "bbo_":
        run.argtypes = [C.POINTER(Cfg), C.POINTER(Inputs), C.POINTER(Metrics), C.POINTER(Detail)]
        lib.bbo_generate_arrivals.argtypes = [C.c_uint64, C.c_double, C.c_uint64, _dp]
    else:
        run.argtypes = [C.POINTER(Cfg), C.POINTER(Metrics), C.POINTER(Detail)]
        lib.bbref_run_arrays.argtypes = [C.POINTER(Cfg), _dp, _dp, C.POINTER(Metrics), C.POINTER(Detail)]
        lib.bbref_run_replicas.argtypes = [C.POINTER(Cfg), C.c_uint64, C.c_uint64, C.c_uint64,
                                           C.c_int, C.POINTER(Metrics), C.POINTER(C.c_double)]
        for f in ("bbref_throughput",):
            getattr(lib, f).restype = C.c_double
            getattr(lib, f).argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double]
        lib.bbref_expected_latency.restype = C.c_double
        lib.bbref_expected_latency.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double,
                                               C.c_double]
        lib.bbref_expected_max_uniform.restype = C.c_double
        lib.bbref_expected_max_uniform.argtypes = [C.c_uint64, C.c_double, C.c_double]
        lib.bbref_uniform_boundaries.argtypes = [C.c_uint64, C.c_double, C.c_double, _dp]
        lib.bbref_exponential_boundaries.argtypes = [C.c_uint64, C.c_double, C.c_uint64, _dp]
        lib.bbref_empirical_boundaries.argtypes = [C.c_uint64, _dp, C.c_uint64, _dp]
    lib.run_fn = run
    return lib


_cache = {}


def oracle():
    if "o" not in _cache:
        _cache["o"] = _load(ORACLE_SO, "bbo_")
    return _cache["o"]


def reference():
    if "r" not in _cache:
        _cache["r"] = _load(REF_SO, "bbref_")
    return _cache["r"]


def have_reference():
    return os.path.exists(REF_SO)


class _Keep:
    """keeps numpy buffers alive while a Cfg points at them"""


def make_cfg(d: dict):
    """dict (SimConfig field names) -> (Cfg, keepalive)"""
    keep = _Keep()
    c = Cfg()
    c.arrival_rate = float(d.get("arrival_rate", math.inf))
    c.n_requests = int(d["n_requests"])
    c.batch_size = int(d.get("batch_size", 1))
    c.n_servers = int(d.get("n_servers", 1))
    c.seed = int(d.get("seed", 0)) & (2**64 - 1)
    c.flush_partial = int(bool(d.get("flush_partial", True)))
    mbw = d.get("max_batch_wait")
    c.has_max_batch_wait = int(mbw is not None)
    c.max_batch_wait = float(mbw) if mbw is not None else 0.0
    if d.get("edges") is not None and len(d["edges"]):
        keep.edges = np.ascontiguousarray(d["edges"], dtype=np.float64)
        c.edges = _ptr(keep.edges, _dp)
        c.n_edges = len(keep.edges)
    c.error_kind = ERR[d.get("error", "perfect")]
    c.p_error = float(d.get("p_error", 0.0))
    if d.get("confusion") is not None:
        keep.conf = np.ascontiguousarray(d["confusion"], dtype=np.float64).ravel()
        c.confusion = _ptr(keep.conf, _dp)
    c.service_kind = SVC[d.get("service", "uniform")]
    c.lo = float(d.get("lo", 1.0))
    c.hi = float(d.get("hi", 2.0))
    c.rate = float(d.get("rate", 1.0))
    c.lin_a = float(d.get("lin_a", 0.0))
    c.lin_b = float(d.get("lin_b", 1.0))
    c.mu = float(d.get("mu", 0.0))
    c.sigma = float(d.get("sigma", 1.0))
    if d.get("table") is not None:
        keep.table = np.ascontiguousarray(d["table"], dtype=np.float64)
        c.table = _ptr(keep.table, _dp)
        c.n_table = len(keep.table)
    return c, keep


def run(lib, d: dict, inputs: dict | None = None, detail: bool = True):
    """Run one simulation; returns (metrics dict, detail dict | None).

    Raises OracleError(code, msg) with the reference's exception category."""
    c, keep = make_cfg(d)
    n = c.n_requests
    k = c.n_edges - 1
    m = Metrics()
    det = None
    out = None
    if detail:
        out = dict(
            req_arrival=np.empty(n), req_service=np.empty(n),
            req_true_bin=np.empty(n, np.uint32), req_pred_bin=np.empty(n, np.uint32),
            req_batch=np.empty(n, np.uint64), req_completion=np.empty(n),
            bat_bin=np.empty(n, np.uint32), bat_size=np.empty(n, np.uint64),
            bat_first=np.empty(n, np.uint64), bat_formed=np.empty(n), bat_start=np.empty(n),
            bat_finish=np.empty(n), bat_service=np.empty(n), members=np.empty(n, np.uint64),
            per_bin_batch_counts=np.zeros(max(k, 1), np.uint64),
        )
        det = Detail()
        for name, t in Detail._fields_:
            setattr(det, name, out[name].ctypes.data_as(t))
    if lib.prefix == "bbo_":
        inp = Inputs()
        if inputs:
            for key in ("arrivals", "services", "u_err"):
                if inputs.get(key) is not None:
                    arr = np.ascontiguousarray(inputs[key], dtype=np.float64)
                    setattr(keep, key, arr)
                    setattr(inp, key, _ptr(arr, _dp))
            if inputs.get("pred_bin") is not None:
                keep.pred = np.ascontiguousarray(inputs["pred_bin"], dtype=np.uint8)
                inp.pred_bin = _ptr(keep.pred, _u8p)
        st = lib.run_fn(C.byref(c), C.byref(inp), C.byref(m), C.byref(det) if det else None)
    elif inputs:  # the reference engine on given arrivals/services (bbref_run_arrays)
        if inputs.get("u_err") is not None or inputs.get("pred_bin") is not None:
            raise ValueError("reference arrays mode draws predictions from the seed's stream 2")
        keep.a = np.ascontiguousarray(inputs["arrivals"], dtype=np.float64)
        keep.s = np.ascontiguousarray(inputs["services"], dtype=np.float64)
        st = lib.bbref_run_arrays(C.byref(c), _ptr(keep.a, _dp), _ptr(keep.s, _dp), C.byref(m),
                                  C.byref(det) if det else None)
    else:
        st = lib.run_fn(C.byref(c), C.byref(m), C.byref(det) if det else None)
    if st != OK:
        raise OracleError(st, lib.last().decode())
    md = m.as_dict()
    if out is not None:
        nb = m.n_batches
        for key in list(out):
            if key.startswith("bat_"):
                out[key] = out[key][:nb]
        out["per_bin_batch_counts"] = out["per_bin_batch_counts"][:k]
        out["members"] = out["members"][: int(out["bat_size"].sum())]
    return md, out


def stream_uniform01(lib, seed, stream_id, n):
    out = np.empty(n)
    lib.stream_uniform01(seed & (2**64 - 1), stream_id, n, out.ctypes.data_as(_dp))
    return out


def acceptance_trace(n=20000, seed=424242):
    """The long-tailed trace of acceptance.cpp:366-375: RandomStream(424242),
    v = min((1-u)^(-1/1.2), 500)."""
    lib = oracle()
    u = np.empty(n)
    lib.bbo_plain_uniform01.argtypes = [C.c_uint64, C.c_uint64, _dp]
    lib.bbo_plain_uniform01(seed, n, u.ctypes.data_as(_dp))
    return np.minimum(np.power(1.0 - u, -1.0 / 1.2), 500.0)


def run_replicas(d: dict, master: int, rep0: int, nrep: int, threads: int):
    """Reference replications on `threads` host threads -> (per-rep metrics list, seconds)."""
    lib = reference()
    c, keep = make_cfg(d)
    arr = (Metrics * nrep)()
    secs = C.c_double()
    st = lib.bbref_run_replicas(C.byref(c), master, rep0, nrep, threads, arr, C.byref(secs))
    if st != OK:
        raise OracleError(st, lib.last().decode())
    return [a.as_dict() for a in arr], secs.value


POINT_FIELDS = ("throughput_mean", "throughput_std", "latency_mean", "latency_std", "latency_p50",
                "latency_p99", "makespan_mean", "busy_fraction_mean", "analytic_throughput",
                "analytic_latency", "analytic_max_throughput")


def run_point(d: dict, k: int, master: int, reps: int) -> dict:
    """The reference's own run_point (experiment.hpp:254-307) on the template
    `d` describes (edges omitted -> derived from k) -> PointResult numbers."""
    lib = reference()
    lib.bbref_run_point.argtypes = [C.POINTER(Cfg), C.c_uint64, C.c_uint64, C.c_uint64, _dp]
    c, keep = make_cfg(d)
    out = np.empty(len(POINT_FIELDS))
    st = lib.bbref_run_point(C.byref(c), k, master, reps, out.ctypes.data_as(_dp))
    if st != OK:
        raise OracleError(st, lib.last().decode())
    return dict(zip(POINT_FIELDS, out.tolist()))


def uniform_boundaries(k, lo, hi):
    out = np.empty(k + 1)
    st = reference().bbref_uniform_boundaries(k, lo, hi, out.ctypes.data_as(_dp))
    if st:
        raise OracleError(st, reference().last().decode())
    return out
