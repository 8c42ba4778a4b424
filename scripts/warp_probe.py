"""One warp-mode launch (C5 shape, reduced replications) for ncu."""
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

import paper_2412_04504_b200 as bb  # noqa: E402

svc = bb.ServiceSpec("lognormal", mu=0.0, sigma=1.0)
t = bb.RunTemplate(arrival_rate=17.0, n_requests=1_000_000, batch_size=64, bins=bb.BinRule(k=16), service=svc)
R = 148 * 16 * 2
rep = torch.zeros(6 * R, dtype=torch.float64, device="cuda")
bb.points_shard_device([t], R, 11, 0, R, rep.data_ptr())
torch.cuda.synchronize()
print(rep.view(6, R)[:, :4])
