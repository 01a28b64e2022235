"""Kernel timeline of one GGN product (torch.profiler): start/end offsets per stream."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
from torch.profiler import profile, ProfilerActivity
m = P.Model(784, (1024, 1024), 10, "relu")
w = P.init_params(m, P.Rng(0)).to_device()
r = P.Rng(1); b = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
X = torch.from_numpy(r.normal(b*784).reshape(b,784).astype(np.float32)).cuda()
y = torch.from_numpy(r.integers(b,10)).cuda()
snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
v = torch.randn(w.dim, device="cuda"); out = torch.empty_like(v)
for _ in range(5): snap.apply(0, v, out)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3): snap.apply(0, v, out)
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
n = len(evs) // 3
ev = evs[n:2 * n]
t0 = ev[0].time_range.start
for e in ev:
    print(f"{e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f} {e.time_range.end - e.time_range.start:7.1f}  "
          f"{getattr(e, 'device_index', '')} {e.name[:70]}")
