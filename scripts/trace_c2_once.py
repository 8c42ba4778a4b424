"""One C2 trace-mode run with bench.py's inputs (reference-generated arrays,
predicted bins given), for ncu captures of the trace pipeline."""
import os
import sys

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
st = torch.cuda.current_stream().cuda_stream
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    m = bb.run_trace_device(cfg, a.data_ptr(), s.data_ptr(), 0, p.data_ptr(), st)
torch.cuda.synchronize()
print(m.makespan == mr["makespan"], m.latency_p99 == mr["latency_p99"])
