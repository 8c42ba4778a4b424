"""C2 trace timing split: device events around the call vs host wall time
(BB_TRACE_MS=1 also prints the pipeline's own first-to-last-kernel time)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import torch  # noqa: E402

import oracle_py as O  # noqa: E402
import paper_2412_04504_b200 as bb  # noqa: E402

n = 10_000_000
lam = 0.95 * bb.throughput(16, 8, 1.0, 20.0)
edges = bb.uniform_boundaries(8, 1.0, 20.0)
mr, dr = O.run(O.reference(), dict(arrival_rate=lam, n_requests=n, batch_size=16, edges=edges.edges,
                                   lo=1.0, hi=20.0, seed=1001, error="symmetric", p_error=0.1))
a = torch.from_numpy(dr["req_arrival"]).cuda()
s = torch.from_numpy(dr["req_service"]).cuda()
p = torch.from_numpy(dr["req_pred_bin"].astype("uint8")).cuda()
cfg = bb.SimConfig(arrival_rate=lam, n_requests=n, batch_size=16, bins=edges)
stream = torch.cuda.Stream()
st = stream.cuda_stream
for _ in range(5):
    m = bb.run_trace_device(cfg, a.data_ptr(), s.data_ptr(), 0, p.data_ptr(), st)
ev, wall = [], []
for _ in range(10):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    m = bb.run_trace_device(cfg, a.data_ptr(), s.data_ptr(), 0, p.data_ptr(), st)
    e1.record(stream)
    torch.cuda.synchronize()
    wall.append((time.perf_counter() - t0) * 1e3)
    ev.append(e0.elapsed_time(e1))
print("events ms", sorted(ev)[5], "wall ms", sorted(wall)[5], "graph", bb.trace_graph_stats(),
      m.makespan == mr["makespan"], m.latency_p99 == mr["latency_p99"])
