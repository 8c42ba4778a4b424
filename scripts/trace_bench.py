"""C2 trace-mode timing only (bench.py's trace leg), for iteration."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2412_04504_b200 as bb  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream()
out = bench.trace_measure(bb, torch, dev, stream)
print(json.dumps(out))
