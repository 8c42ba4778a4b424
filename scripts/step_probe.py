"""Where the bench step's time goes outside gen_kernel: device events around
the shard call and the reduce, host time of each call, at two sizes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2412_04504_b200 as bb  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(stream)
sptr = stream.cuda_stream
pts = bench.sweep_points(100000)
tpl = [bb.RunTemplate(arrival_rate=p["lam"], n_requests=p["n"], batch_size=p["B"], bins=bb.BinRule(k=p["k"]),
                      service=bb.ServiceSpec("linear", 1.0, 1024.0, intercept=bench.A_INTERCEPT,
                                             slope=bench.B_SLOPE)) for p in pts]
sampler = bench.ClockSampler(0) if os.environ.get("PROBE_CLOCKS") else None
if sampler:
    sampler.__enter__()
for R in [int(x) for x in sys.argv[1:]] or [2000, 10000]:
    block = torch.empty(6 * len(tpl) * R, dtype=torch.float64, device=dev)
    for it in range(4):
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        t0 = time.perf_counter()
        ev[0].record(stream)
        bb.points_shard_local_device(tpl, R, 1234, 0, R, block.data_ptr(), sptr)
        t1 = time.perf_counter()
        ev[1].record(stream)
        bb.points_reduce_gathered_device(tpl, R, 1, block.data_ptr(), sptr)
        t2 = time.perf_counter()
        ev[2].record(stream)
        torch.cuda.synchronize()
        print(f"R={R} it={it} step_ms={ev[0].elapsed_time(ev[2]):.2f} shard_dev_ms={ev[0].elapsed_time(ev[1]):.2f} "
              f"reduce_dev_ms={ev[1].elapsed_time(ev[2]):.2f} kernel_ms={bb.last_kernel_ms()[0]:.2f} "
              f"host_shard_ms={(t1-t0)*1e3:.2f} host_reduce_ms={(t2-t1)*1e3:.2f}", flush=True)
if sampler:
    sampler.__exit__(None, None, None)
