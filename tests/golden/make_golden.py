"""Generate the golden fixtures in tests/golden/*.npz from the REFERENCE itself.

Runs /root/reference's engine (oracle/_ref/libbbref.so, built by
`make -C oracle` from the reference headers in place) on small configurations
and stores, per fixture:

  config      json of the SimConfig fields (oracle_py.make_cfg vocabulary)
  arrivals, services, u_err   the request streams the reference drew
                              (u_err = RandomStream::derive(seed, 2) replayed)
  req_* / bat_* / members     the reference's Request / BatchRecord vectors
  metrics     json of SimMetrics

Usage:  python tests/golden/make_golden.py      (needs /root/reference)
"""
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import oracle_py as O  # noqa: E402


def edges(k, lo=1.0, hi=20.0):
    return O.uniform_boundaries(k, lo, hi).tolist()


CAP8 = 128 / 10.5  # not used; capacity of B=16,k=8 below
LAM_C2 = 0.95 * 1.385550  # 0.95 x throughput(16, 8, 1, 20)

FIXTURES = {
    "c2_poisson_perfect": dict(arrival_rate=LAM_C2, n_requests=4000, batch_size=16,
                               edges=edges(8), lo=1.0, hi=20.0, seed=1001),
    "c2_poisson_symmetric": dict(arrival_rate=LAM_C2, n_requests=4000, batch_size=16,
                                 edges=edges(8), lo=1.0, hi=20.0, seed=1001,
                                 error="symmetric", p_error=0.1),
    "c2_load099": dict(arrival_rate=0.99 * 1.385550, n_requests=8000, batch_size=16,
                       edges=edges(8), lo=1.0, hi=20.0, seed=7),
    "overload_flush_sym": dict(arrival_rate=math.inf, n_requests=1000, batch_size=8,
                               edges=edges(3), lo=1.0, hi=20.0, seed=5, error="symmetric",
                               p_error=0.2),
    "overload_noflush": dict(arrival_rate=math.inf, n_requests=1003, batch_size=16,
                             edges=edges(5), lo=1.0, hi=20.0, seed=9, flush_partial=False),
    "poisson_noflush": dict(arrival_rate=4.0, n_requests=640, batch_size=8, edges=edges(2),
                            lo=1.0, hi=20.0, seed=17, flush_partial=False),
    "confusion": dict(arrival_rate=3.0, n_requests=2000, batch_size=8, edges=edges(3), lo=1.0,
                      hi=20.0, seed=11, error="confusion",
                      confusion=[[0.7, 0.25, 0.05], [0.15, 0.7, 0.15], [0.02, 0.28, 0.7]]),
    "exponential": dict(arrival_rate=0.8, n_requests=3000, batch_size=8,
                        edges=[0.0, 1.0, 2.5, math.inf], seed=21, service="exponential",
                        rate=0.2),
    "kat_1526_k1": dict(arrival_rate=math.inf, n_requests=4, batch_size=2, edges=[1.0, 6.0],
                        seed=2, service="trace_cyclic", table=[1.0, 5.0, 2.0, 6.0]),
    "kat_1526_k2": dict(arrival_rate=math.inf, n_requests=4, batch_size=2,
                        edges=[1.0, 3.5, 6.0], seed=2, service="trace_cyclic",
                        table=[1.0, 5.0, 2.0, 6.0]),
    "kat_16_mixed": dict(arrival_rate=math.inf, n_requests=8, batch_size=2, edges=[1.0, 6.0],
                         seed=1, service="trace_cyclic", table=[1.0, 6.0]),
    "kat_16_split": dict(arrival_rate=math.inf, n_requests=8, batch_size=2,
                         edges=[1.0, 3.5, 6.0], seed=1, service="trace_cyclic",
                         table=[1.0, 6.0]),
}


def jsonable(d):
    out = {}
    for k, v in d.items():
        if isinstance(v, np.ndarray):
            v = v.tolist()
        if isinstance(v, float) and math.isinf(v):
            v = "inf"
        if isinstance(v, list):
            v = ["inf" if isinstance(x, float) and math.isinf(x) else x for x in v]
        out[k] = v
    return out


def main():
    ref = O.reference()
    for name, cfg in FIXTURES.items():
        m, d = O.run(ref, cfg)
        n = cfg["n_requests"]
        draws = cfg.get("error") == "confusion" or (
            cfg.get("error") == "symmetric" and len(cfg["edges"]) > 2 and cfg["p_error"] > 0)
        u = O.stream_uniform01(ref, cfg["seed"], 2, n) if draws else np.zeros(0)
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"),
            config=json.dumps(jsonable(cfg)), metrics=json.dumps(m),
            arrivals=d["req_arrival"], services=d["req_service"], u_err=u,
            req_true_bin=d["req_true_bin"].astype(np.uint8),
            req_pred_bin=d["req_pred_bin"].astype(np.uint8),
            req_batch=d["req_batch"], req_completion=d["req_completion"],
            bat_bin=d["bat_bin"].astype(np.uint8), bat_size=d["bat_size"],
            bat_first=d["bat_first"], bat_formed=d["bat_formed"], bat_start=d["bat_start"],
            bat_finish=d["bat_finish"], bat_service=d["bat_service"], members=d["members"],
            per_bin=d["per_bin_batch_counts"])
        print(f"{name}: n={n} batches={m['n_batches']} makespan={m['makespan']!r}")


if __name__ == "__main__":
    main()
