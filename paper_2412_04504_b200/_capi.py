"""ctypes declarations of include/binbatch_b200.h.

The shared library is required: importing this module without it raises
ImportError -- there is no CPU fallback anywhere in the package.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BB_LIB_PATH") or os.path.join(PKG, "libbinbatch_b200.so")

BB_OK, BB_EINVAL, BB_EDOMAIN, BB_ERUNTIME, BB_ECUDA, BB_EUNSUPPORTED = range(6)
BB_MAX_BINS = 64
BB_TRACE_MAX_BINS = 32
BB_NO_BATCH = 0xFFFFFFFF
BB_REP_FIELDS = 6

SVC = {"uniform": 0, "exponential": 1, "empirical": 2, "trace_cyclic": 3, "trace_resample": 4,
       "linear": 6, "lognormal": 7}
ERR = {"perfect": 0, "symmetric": 1, "confusion": 2}
RNG = {"philox": 0, "reference": 1}
KIND = {"uniform": 0, "exponential": 1, "trace": 2, "linear": 3, "lognormal": 4}
AXIS = {"lambda": 0, "k": 1, "B": 2, "p_e": 3, "n_servers": 4}

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)


class SimConfigC(C.Structure):
    _fields_ = [
        ("arrival_rate", C.c_double), ("n_requests", C.c_uint64), ("batch_size", C.c_uint64),
        ("n_servers", C.c_uint64), ("seed", C.c_uint64), ("flush_partial", C.c_int32),
        ("has_max_batch_wait", C.c_int32), ("max_batch_wait", C.c_double), ("edges", _dp),
        ("n_edges", C.c_uint64), ("error_kind", C.c_int32), ("service_kind", C.c_int32),
        ("p_error", C.c_double), ("confusion", _dp), ("lo", C.c_double), ("hi", C.c_double),
        ("rate", C.c_double), ("lin_a", C.c_double), ("lin_b", C.c_double), ("mu", C.c_double),
        ("sigma", C.c_double), ("table", _dp), ("n_table", C.c_uint64), ("rng", C.c_int32),
        ("device", C.c_int32), ("confusion_k", C.c_uint64),
    ]


class SimMetricsC(C.Structure):
    _fields_ = [
        ("throughput", C.c_double), ("makespan", C.c_double), ("latency_mean", C.c_double),
        ("latency_p50", C.c_double), ("latency_p99", C.c_double),
        ("server_busy_fraction", C.c_double), ("n_completed", C.c_uint64),
        ("n_batches", C.c_uint64), ("k", C.c_uint64),
        ("per_bin_batch_counts", C.c_uint64 * BB_MAX_BINS), ("busy_time", C.c_double),
        ("latency_sum", C.c_double),
    ]


class SimDetailC(C.Structure):
    _fields_ = [
        ("req_arrival", _dp), ("req_service", _dp), ("req_true_bin", _u8p),
        ("req_pred_bin", _u8p), ("req_batch", _u32p), ("req_completion", _dp),
        ("batch_capacity", C.c_uint64), ("bat_bin", _u8p), ("bat_size", _u32p),
        ("bat_first", _u32p), ("bat_formed", _dp), ("bat_start", _dp), ("bat_finish", _dp),
        ("bat_service", _dp), ("members", _u32p),
    ]


class TraceInC(C.Structure):
    _fields_ = [("arrivals", _dp), ("services", _dp), ("u_err", _dp), ("pred_bin", _u8p)]


class PointResultC(C.Structure):
    _fields_ = [
        ("arrival_rate", C.c_double), ("k", C.c_uint64), ("batch_size", C.c_uint64),
        ("n_servers", C.c_uint64), ("error_kind", C.c_int32), ("p_error", C.c_double),
        ("n_requests", C.c_uint64), ("replications", C.c_uint64),
        ("throughput_mean", C.c_double), ("throughput_std", C.c_double),
        ("latency_mean", C.c_double), ("latency_std", C.c_double),
        ("latency_p50", C.c_double), ("latency_p99", C.c_double),
        ("makespan_mean", C.c_double), ("busy_fraction_mean", C.c_double),
        ("analytic_throughput", C.c_double), ("analytic_latency", C.c_double),
        ("analytic_max_throughput", C.c_double),
    ]


class RunTemplateC(C.Structure):
    _fields_ = [
        ("arrival_rate", C.c_double), ("n_requests", C.c_uint64), ("batch_size", C.c_uint64),
        ("n_servers", C.c_uint64), ("flush_partial", C.c_int32), ("has_max_batch_wait", C.c_int32),
        ("max_batch_wait", C.c_double), ("service", C.c_int32), ("trace_cyclic", C.c_int32),
        ("min_time", C.c_double), ("max_time", C.c_double), ("rate", C.c_double),
        ("lin_a", C.c_double), ("lin_b", C.c_double), ("mu", C.c_double), ("sigma", C.c_double),
        ("trace_times", _dp), ("n_trace", C.c_uint64), ("k", C.c_uint64), ("edges", _dp),
        ("n_edges", C.c_uint64), ("error_kind", C.c_int32), ("p_error", C.c_double),
        ("confusion", _dp), ("confusion_k", C.c_uint64),
    ]


class SweepAxisC(C.Structure):
    _fields_ = [("param", C.c_int32), ("values", _dp), ("n_values", C.c_uint64)]


class ExperimentSpecC(C.Structure):
    _fields_ = [("base", RunTemplateC), ("axes", SweepAxisC * 2), ("n_axes", C.c_uint64),
                ("replications", C.c_uint64), ("seed", C.c_uint64), ("rng", C.c_int32),
                ("name", C.c_char_p)]


# every symbol include/binbatch_b200.h declares (checked by tests/test_capi_symbols.py)
EXPORTS = [
    "bb_last_error", "bb_abi_version", "bb_device_info", "bb_run_simulation",
    "bb_run_simulation_detailed", "bb_replay_trace", "bb_replay_trace_detailed", "bb_run_trace",
    "bb_run_trace_device", "bb_replication_seed", "bb_run_point", "bb_run_experiment",
    "bb_sweep_shard_device", "bb_sweep_reduce_device", "bb_experiment_points",
    "bb_uniform_boundaries", "bb_exponential_boundaries", "bb_empirical_boundaries",
    "bb_analytic_throughput", "bb_analytic_latency", "bb_philox4x32_10", "bb_launch_count",
    "bb_last_kernel_ms", "bb_points_shard_device", "bb_run_points", "bb_points_reduce_device", "bb_transfer_bytes",
    "bb_exponential_variates", "bb_set_generated_quantiles", "bb_template_edges",
    "bb_service_of_keys", "bb_expected_service_time", "bb_throughput", "bb_max_throughput",
    "bb_min_bins_for_throughput", "bb_expected_latency", "bb_exponential_service_bound",
    "bb_harmonic_number", "bb_assign_bin", "bb_brute_force_boundaries",
    "bb_points_shard_local_device", "bb_points_reduce_gathered_device", "bb_set_devices",
    "bb_trace_graph_stats",
]


def load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2412_04504_b200/build.py` "
            "(the engine has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    lib.bb_last_error.restype = C.c_char_p
    lib.bb_abi_version.restype = C.c_int
    lib.bb_device_info.argtypes = [C.c_int32, C.c_char_p, C.c_size_t, P(C.c_int32), P(C.c_int32),
                                   P(C.c_int32)]
    lib.bb_run_simulation.argtypes = [P(SimConfigC), P(SimMetricsC)]
    lib.bb_run_simulation_detailed.argtypes = [P(SimConfigC), P(SimMetricsC), P(SimDetailC)]
    lib.bb_replay_trace.argtypes = [P(SimConfigC), _dp, C.c_uint64, P(SimMetricsC)]
    lib.bb_replay_trace_detailed.argtypes = [P(SimConfigC), _dp, C.c_uint64, P(SimMetricsC),
                                             P(SimDetailC)]
    lib.bb_run_trace.argtypes = [P(SimConfigC), P(TraceInC), P(SimMetricsC), P(SimDetailC)]
    lib.bb_run_trace_device.argtypes = [P(SimConfigC), P(TraceInC), P(SimMetricsC),
                                        P(SimDetailC), C.c_void_p]
    lib.bb_replication_seed.restype = C.c_uint64
    lib.bb_replication_seed.argtypes = [C.c_uint64, C.c_uint64]
    lib.bb_run_point.argtypes = [P(RunTemplateC), C.c_uint64, C.c_uint64, P(PointResultC)]
    lib.bb_run_experiment.argtypes = [P(ExperimentSpecC), C.c_uint, P(PointResultC), C.c_uint64,
                                      P(C.c_uint64)]
    lib.bb_sweep_shard_device.argtypes = [P(ExperimentSpecC), C.c_uint64, C.c_uint64, C.c_void_p,
                                          C.c_void_p]
    lib.bb_sweep_reduce_device.argtypes = [P(ExperimentSpecC), C.c_void_p, P(PointResultC),
                                           C.c_void_p]
    lib.bb_points_shard_device.argtypes = [P(RunTemplateC), C.c_uint64, C.c_uint64, C.c_uint64,
                                           C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p]
    lib.bb_run_points.argtypes = [P(RunTemplateC), C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32,
                                  P(PointResultC)]
    lib.bb_points_reduce_device.argtypes = [P(RunTemplateC), C.c_uint64, C.c_uint64, C.c_void_p,
                                            P(PointResultC), C.c_void_p]
    lib.bb_points_shard_local_device.argtypes = [P(RunTemplateC), C.c_uint64, C.c_uint64, C.c_uint64,
                                                 C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p]
    lib.bb_points_reduce_gathered_device.argtypes = [P(RunTemplateC), C.c_uint64, C.c_uint64,
                                                     C.c_uint32, C.c_void_p, P(PointResultC),
                                                     C.c_void_p]
    lib.bb_set_devices.argtypes = [P(C.c_int32), C.c_uint32]
    lib.bb_experiment_points.argtypes = [P(ExperimentSpecC), P(C.c_uint64)]
    lib.bb_uniform_boundaries.argtypes = [C.c_uint64, C.c_double, C.c_double, _dp]
    lib.bb_exponential_boundaries.argtypes = [C.c_uint64, C.c_double, C.c_uint64, _dp]
    lib.bb_empirical_boundaries.argtypes = [C.c_uint64, _dp, C.c_uint64, _dp]
    lib.bb_analytic_throughput.restype = C.c_double
    lib.bb_analytic_throughput.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double]
    lib.bb_analytic_latency.restype = C.c_double
    lib.bb_analytic_latency.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_double]
    lib.bb_philox4x32_10.argtypes = [P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]
    lib.bb_exponential_variates.restype = C.c_int
    lib.bb_exponential_variates.argtypes = [P(C.c_uint64), C.c_uint64, C.c_int32, _dp]
    lib.bb_transfer_bytes.argtypes = [P(C.c_uint64), P(C.c_uint64), C.c_int]
    lib.bb_launch_count.restype = C.c_uint64
    lib.bb_launch_count.argtypes = [C.c_int]
    lib.bb_last_kernel_ms.restype = C.c_double
    lib.bb_last_kernel_ms.argtypes = [P(C.c_char_p)]
    lib.bb_trace_graph_stats.restype = None
    lib.bb_trace_graph_stats.argtypes = [P(C.c_uint64), P(C.c_uint64), C.c_int]
    lib.bb_template_edges.argtypes = [P(RunTemplateC), _dp, C.c_uint64, P(C.c_uint64)]
    lib.bb_service_of_keys.argtypes = [P(RunTemplateC), P(C.c_uint64), C.c_uint64, _dp]
    for f in ("bb_expected_service_time", "bb_throughput"):
        getattr(lib, f).argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double, _dp]
    lib.bb_max_throughput.argtypes = [C.c_uint64, C.c_double, C.c_double, _dp]
    lib.bb_min_bins_for_throughput.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_double,
                                               P(C.c_uint64)]
    lib.bb_expected_latency.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double,
                                        C.c_double, _dp]
    lib.bb_exponential_service_bound.argtypes = [C.c_uint64, C.c_uint64, C.c_double, _dp]
    lib.bb_harmonic_number.argtypes = [C.c_uint64, _dp]
    lib.bb_assign_bin.argtypes = [_dp, C.c_uint64, C.c_double, P(C.c_uint64)]
    lib.bb_brute_force_boundaries.argtypes = [C.c_uint64, C.c_int32, C.c_double, C.c_double,
                                              C.c_uint64, C.c_uint64, _dp]
    lib.bb_set_generated_quantiles.restype = C.c_int
    lib.bb_set_generated_quantiles.argtypes = [C.c_int]
    return lib
