"""Kernel timeline of one linearization (make_snapshot) at C3 (torch.profiler)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
from torch.profiler import profile, ProfilerActivity
m = P.Model(784, (1024, 1024), 10, "relu")
w = P.init_params(m, P.Rng(0)).to_device()
r = P.Rng(1); b = 8192
X = torch.from_numpy(r.normal(b*784).reshape(b,784).astype(np.float32)).cuda()
y = torch.from_numpy(r.integers(b,10)).cuda()
batch = P.Batch(X, y, "ce")
for _ in range(3):
    P.make_snapshot("ggn_ce", m, w, batch).close()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s = P.make_snapshot("ggn_ce", m, w, batch)
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
for e in evs:
    print(f"{e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f} {e.time_range.end - e.time_range.start:7.1f}  {e.name[:80]}")
