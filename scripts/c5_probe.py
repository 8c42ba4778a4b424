"""C5-shape sample (bench.c5_measure) on its own, for iteration."""
import json
import sys
import time

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2412_04504_b200 as bb  # noqa: E402

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
t0 = time.perf_counter()
out = bench.c5_measure(bb, torch, stream)
print(json.dumps(out), "wall", time.perf_counter() - t0)
