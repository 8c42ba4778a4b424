import sys, os, math
sys.path[:0] = [os.getcwd(), os.getcwd() + "/oracle", os.getcwd() + "/tests"]
import numpy as np
import oracle_py as O
import paper_2412_04504_b200 as bb
from test_gpu_quantiles import replica_streams, kernel_rep_metrics
lam, n, B, k, S, flush, pe, W = (0.8, 20000, 16, 4, 1, True, 0.0, 6.0)
t = bb.RunTemplate(arrival_rate=lam, n_requests=n, batch_size=B, n_servers=S, flush_partial=flush,
                   bins=bb.BinRule(k=k), service=bb.ServiceSpec("uniform", 1.0, 20.0), max_batch_wait=W)
got = kernel_rep_metrics(t, 40, 4711)
edges = bb.uniform_boundaries(k, 1.0, 20.0).edges
for r in (0, 1, 2, 3):
    a, s, u = replica_streams(4711, r, n, lam, 1.0, 20.0, False)
    cfg = dict(arrival_rate=lam, n_requests=n, batch_size=B, n_servers=S, flush_partial=flush, edges=edges,
               lo=1.0, hi=20.0, service="arrays", max_batch_wait=W)
    m, d = O.run(O.oracle(), cfg, inputs=dict(arrivals=a, services=s), detail=True)
    lat = np.sort(d["req_completion"] - d["req_arrival"])
    print(r, "kernel", got[:, r])
    print(r, "oracle", m["throughput"], m["latency_mean"], m["latency_p50"], m["latency_p99"], m["makespan"], "lat min/max", lat[0], lat[-1])
    print("   rank of kernel p50", np.searchsorted(lat, got[2, r]), "of", len(lat), "timer batches", int((d["bat_size"] < B).sum()), "of", len(d["bat_size"]))
