"""Small trace-mode runs for compute-sanitizer (memcheck / racecheck): the
direct pipeline, its graph capture and a replay, given and drawn predictions."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import torch  # noqa: E402

import oracle_py as O  # noqa: E402
import paper_2412_04504_b200 as bb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000
lam = 0.95 * bb.throughput(16, 8, 1.0, 20.0)
edges = bb.uniform_boundaries(8, 1.0, 20.0)
cfg_d = dict(arrival_rate=lam, n_requests=n, batch_size=16, edges=edges.edges, lo=1.0, hi=20.0,
             seed=7, error="symmetric", p_error=0.1)
mr, dr = O.run(O.oracle(), cfg_d)
a = torch.from_numpy(dr["req_arrival"]).cuda()
s = torch.from_numpy(dr["req_service"]).cuda()
p = torch.from_numpy(dr["req_pred_bin"].astype("uint8")).cuda()
cfg = bb.SimConfig(arrival_rate=lam, n_requests=n, batch_size=16, bins=edges)
st = torch.cuda.Stream()
ok = True
for _ in range(3):  # direct, capture, replay
    m = bb.run_trace_device(cfg, a.data_ptr(), s.data_ptr(), 0, p.data_ptr(), st.cuda_stream)
    ok &= m.makespan == mr["makespan"] and m.latency_p99 == mr["latency_p99"]
res = bb.run_trace(bb.SimConfig(arrival_rate=lam, n_requests=n, batch_size=16, bins=edges,
                                error_model=bb.Symmetric(0.1)),
                   dr["req_arrival"], dr["req_service"], u_err=O.stream_uniform01(O.oracle(), 7, 2, n),
                   detailed=True)
ok &= res.metrics.makespan == mr["makespan"]
print("sanitize trace ok" if ok else "MISMATCH", bb.trace_graph_stats())
