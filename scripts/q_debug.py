import sys, os, math
sys.path[:0] = [os.getcwd(), os.getcwd() + "/oracle", os.getcwd() + "/tests"]
import numpy as np
import oracle_py as O
import paper_2412_04504_b200 as bb
from test_gpu_quantiles import replica_streams, kernel_rep_metrics
for case in [(0.9, 20000, 8, 4, 1, True, 0.0), (0.3, 20000, 8, 4, 1, True, 0.0), (0.3, 2000, 8, 1, 1, True, 0.0)]:
    lam, n, B, k, S, flush, pe = case
    lo, hi, master, reps = 1.0, 20.0, 4711, 40
    t = bb.RunTemplate(arrival_rate=lam, n_requests=n, batch_size=B, n_servers=S, flush_partial=flush,
                       bins=bb.BinRule(k=k), service=bb.ServiceSpec("uniform", lo, hi))
    got = kernel_rep_metrics(t, reps, master)
    edges = bb.uniform_boundaries(k, lo, hi).edges
    r = 0
    a, s, u = replica_streams(master, r, n, lam, lo, hi, False)
    cfg = dict(arrival_rate=lam, n_requests=n, batch_size=B, n_servers=S, flush_partial=flush, edges=edges, lo=lo, hi=hi)
    m, d = O.run(O.oracle(), cfg, inputs=dict(arrivals=a, services=s), detail=True)
    lat = np.sort(d["req_completion"] - d["req_arrival"])
    print(case)
    print(" kernel thr lat p50 p99 mk busy:", got[:, r])
    print(" oracle:", m["throughput"], m["latency_mean"], m["latency_p50"], m["latency_p99"], m["makespan"], m["server_busy_fraction"])
    for v in got[2:4, r]:
        idx = np.searchsorted(lat, v)
        print("  value", v, "rank in oracle lat", idx, "present", idx < len(lat) and lat[idx] == v, "of", len(lat), "min/max", lat[0], lat[-1])
