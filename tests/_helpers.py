"""Shared helpers for the parity tests (golden fixtures, comparisons)."""
import glob
import json
import math
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

REQ_KEYS = ("req_true_bin", "req_pred_bin", "req_batch", "req_completion")
BAT_KEYS = ("bat_bin", "bat_size", "bat_first", "bat_formed", "bat_start", "bat_finish",
            "bat_service")


def _unjson(v):
    if v == "inf":
        return math.inf
    if isinstance(v, list):
        return [_unjson(x) for x in v]
    return v


def fixture_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_fixture(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    cfg = {k: _unjson(v) for k, v in json.loads(str(z["config"])).items()}
    metrics = json.loads(str(z["metrics"]))
    arrays = {k: z[k] for k in z.files if k not in ("config", "metrics")}
    return cfg, metrics, arrays


def same_bits(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        return False
    if a.dtype.kind == "f":
        return np.array_equal(a.view(np.uint64), b.astype(np.float64).view(np.uint64))
    return np.array_equal(a.astype(np.int64), b.astype(np.int64))


def sum_tol(n, total_abs):
    """Bound for a reassociated fp64 sum vs the reference's sequential sum."""
    return 2.0 * n * 2.0**-53 * total_abs + 1e-300
