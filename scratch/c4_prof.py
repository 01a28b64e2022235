"""Kernel-time breakdown of one warm C4 planned step (torch.profiler)."""
import sys, collections; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
from torch.profiler import profile, ProfilerActivity
b = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
m = P.Model(3072, (2048, 2048), 10, "relu")
w = P.init_params(m, P.Rng(0)).to_device()
r = P.Rng(1); X = torch.from_numpy(r.normal(b*3072).reshape(b,3072).astype(np.float32)).cuda(); y = torch.from_numpy(r.integers(b,10)).cuda()
batch = P.Batch(X, y, "ce")
meth = P.make("egn_ce", m); st = meth.init(w, 0)
w1, st, info = meth.step(w, batch, st); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); w1, st, info = meth.step(w, batch, st); e1.record(); torch.cuda.synchronize()
print(f"warm step {e0.elapsed_time(e1):.1f} ms")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    w1, st, info = meth.step(w, batch, st); torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        agg[e.name[:60]][0] += 1; agg[e.name[:60]][1] += e.time_range.end - e.time_range.start
for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
    print(f"{t/1e3:8.2f} ms {c:6d}  {n}")
