"""The warp-per-replication quantile kernel (bb_genw_kernel.cuh, chosen for
long replications) against the lane-per-replication kernel: every
per-replication output (throughput, latency_mean, p50, p99, makespan, busy)
bit-identical, across service kinds, error models, flush, ragged lengths and
bin counts up to 32.  (The lane kernel is pinned to the reference through
the oracle in test_gpu_quantiles.py.)"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, %r)
import paper_2412_04504_b200 as bb
U = lambda: bb.ServiceSpec("uniform", 1.0, 20.0)
cases = [
    dict(arrival_rate=17.0, n_requests=20000, batch_size=64, bins=bb.BinRule(k=16),
         service=bb.ServiceSpec("lognormal", mu=0.0, sigma=1.0)),
    dict(arrival_rate=0.9, n_requests=20000, batch_size=16, bins=bb.BinRule(k=8), flush_partial=False,
         service=bb.ServiceSpec("linear", 1.0, 1024.0, intercept=0.5, slope=0.03)),
    dict(arrival_rate=0.7, n_requests=777, batch_size=8, bins=bb.BinRule(k=4), service=U(),
         error=bb.ErrorSpec("symmetric", 0.1)),
    dict(arrival_rate=0.25, n_requests=3001, batch_size=4, bins=bb.BinRule(k=3),
         service=bb.ServiceSpec("exponential", rate=1.0)),
    dict(arrival_rate=0.09, n_requests=500, batch_size=1, bins=bb.BinRule(k=1), service=U()),
    dict(arrival_rate=1.2, n_requests=9000, batch_size=32, bins=bb.BinRule(k=32), service=U(),
         error=bb.ErrorSpec("symmetric", 0.3)),
    dict(arrival_rate=0.5, n_requests=5000, batch_size=8, bins=bb.BinRule(k=5), flush_partial=False,
         service=bb.ServiceSpec("trace", trace_times=[1.0, 2.5, 3.0, 7.5, 9.0, 12.0, 20.0], trace_mode="cyclic")),
]
out = []
R = 64
for c in cases:
    t = bb.RunTemplate(**c)
    rep = torch.zeros(6 * R, dtype=torch.float64, device="cuda")
    bb.points_shard_device([t], R, 20241017, 0, R, rep.data_ptr())
    torch.cuda.synchronize()
    out.append(rep.cpu().numpy().view(np.uint64).tolist())
print(json.dumps(out))
""" % ROOT


def _run(mode):
    env = dict(os.environ, BB_WARP_MODE=mode)
    r = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_warp_kernel_equals_lane_kernel_bit_for_bit():
    lane, warp = _run("0"), _run("1")
    assert len(lane) == len(warp)
    for i, (a, b) in enumerate(zip(lane, warp)):
        assert a == b, f"case {i}: warp-per-replication results differ from the lane kernel"
