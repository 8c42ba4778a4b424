"""Small generated-mode runs (lane kernel with quantiles; BB_WARP_MODE=1 for
the warp kernel) for compute-sanitizer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_04504_b200 as bb  # noqa: E402

svc = bb.ServiceSpec("lognormal", mu=0.0, sigma=1.0)
t = bb.RunTemplate(arrival_rate=15.0, n_requests=int(sys.argv[1]) if len(sys.argv) > 1 else 5000,
                   batch_size=64, bins=bb.BinRule(k=16), service=svc)
p = bb.run_point(t, 3, 64)
print("gen ok", p.throughput_mean, p.latency_p50, p.latency_p99)
