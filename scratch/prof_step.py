"""Kernel-time breakdown + GPU idle time of C3 planned steps (torch.profiler / CUPTI)."""
import sys, os, collections
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2603_25976_b200 as P
from torch.profiler import profile, ProfilerActivity

dev = torch.device("cuda", 0)
model = P.Model(bench.DIMS[0], bench.DIMS[1:-1], bench.DIMS[-1], "relu")
meth = P.assemble(bench.spec_c3(), model)
w = P.init_params(model, P.Rng(0)).to_device(dev)
hb = bench.make_batches(4, bench.GLOBAL_B, 0, 1)
db = [P.Batch(torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev), "ce", global_size=bench.GLOBAL_B) for X, y in hb]
st = meth.init(w, 0)
for i in range(5):
    w, st, info = meth.step(w, db[i % 4], st)
torch.cuda.synchronize()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 10
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(N):
        w, st, info = meth.step(w, db[i % 4], st)
    e1.record(); torch.cuda.synchronize()
wall = e0.elapsed_time(e1) / N
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
agg = collections.defaultdict(lambda: [0, 0.0])
spans = []
for e in evs:
    name = e.name
    agg[name][0] += 1
    agg[name][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    spans.append((e.time_range.start, e.time_range.end))
spans.sort()
busy = 0.0; cur_s, cur_e = None, None
for s, e in spans:
    if cur_e is None or s > cur_e:
        if cur_e is not None: busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
if cur_e is not None: busy += cur_e - cur_s
tot = sum(v[1] for v in agg.values())
print(f"step {wall:.3f} ms (events), kernel busy {busy/1000/N:.3f} ms/step, kernel sum {tot/1000/N:.3f} ms/step")
for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"{t/1000/N:8.3f} ms/step  {n/N:6.1f}/step  {t/n:8.1f} us  {name[:110]}")

# gaps between consecutive kernels (GPU idle), largest first, for one step in the middle
ev = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs), key=lambda t: t[0])
gaps = []
for (s0, e0, n0), (s1, e1, n1) in zip(ev, ev[1:]):
    if s1 - e0 > 15:
        gaps.append((s1 - e0, n0[:50], n1[:50]))
gaps.sort(reverse=True)
tot_gap = sum(g[0] for g in gaps)
print(f"gaps > 15 us: {len(gaps)/N:.1f}/step, {tot_gap/1000/N:.3f} ms/step")
import collections as _c
agg2 = _c.defaultdict(lambda: [0, 0.0])
for g, a, b in gaps:
    agg2[(a, b)][0] += 1
    agg2[(a, b)][1] += g
for (a, b), (n, t) in sorted(agg2.items(), key=lambda kv: -kv[1][1])[:15]:
    print(f"{t/1000/N:7.3f} ms/step {n/N:5.1f}/step  after {a}  before {b}")
