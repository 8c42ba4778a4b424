import sys, os, math
sys.path[:0] = [os.getcwd(), os.getcwd() + "/oracle", os.getcwd() + "/tests"]
import numpy as np
import paper_2412_04504_b200 as bb
from test_gpu_quantiles import replica_streams
lam, n = 0.3, 2000
cfg = bb.SimConfig(arrival_rate=lam, n_requests=n, batch_size=8, bins=bb.uniform_boundaries(1, 1.0, 20.0),
                   service=bb.Uniform(1.0, 20.0), seed=bb.replication_seed(4711, 0))
res = bb.run_simulation_detailed(cfg)
a, s, u = replica_streams(4711, 0, n, lam, 1.0, 20.0, False)
ra = np.asarray(res.requests["arrival"]); rs = np.asarray(res.requests["service"])
print("arr first", ra[:4], a[:4]); print("svc first", rs[:4], s[:4])
print("max rel arr diff", np.max(np.abs(ra - a) / a), "svc equal", np.array_equal(rs, s))
