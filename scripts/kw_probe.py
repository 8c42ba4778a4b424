"""Multi-server trace timing (Philox streams materialised on the device, then the trace pipeline)."""
import sys
import time

sys.path.insert(0, "/root/repo")
import paper_2412_04504_b200 as bb  # noqa: E402

for S, load in ((1, 0.5), (4, 0.5), (4, 1.2), (64, 0.5)):
    n, B, k = 10_000_000, 16, 8
    lam = load * S * bb.throughput(B, k, 1.0, 20.0)
    cfg = bb.SimConfig(arrival_rate=lam, n_requests=n, batch_size=B, bins=bb.uniform_boundaries(k, 1.0, 20.0),
                       service=bb.Uniform(1.0, 20.0), n_servers=S, seed=7, rng="philox")
    bb.run_simulation(cfg)
    t0 = time.perf_counter()
    m = bb.run_simulation(cfg)
    print(f"S={S} load={load}: {1e3 * (time.perf_counter() - t0):.2f} ms wall (incl. draws)  throughput={m.throughput:.5g}")
