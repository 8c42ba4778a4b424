"""One C2-sized trace-mode run (10^7 requests, k=8, B=16) for profiling."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_04504_b200 as bb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
lam = 0.95 * bb.throughput(16, 8, 1.0, 20.0)
cfg = bb.SimConfig(arrival_rate=lam, n_requests=n, batch_size=16,
                   bins=bb.uniform_boundaries(8, 1.0, 20.0), service=bb.Uniform(1.0, 20.0),
                   error_model=bb.Symmetric(0.1), seed=1001, rng="philox")
m = bb.run_simulation(cfg)
print(m.throughput, m.latency_mean, m.latency_p99, bb.last_kernel_ms())
