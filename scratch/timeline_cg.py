"""Kernel timeline of one CG iteration inside a C3 planned step (torch.profiler; PDL
inflates durations, the end offsets are meaningful): the kernels between two k_cg_pap."""
import sys
sys.path.insert(0, ".")
import torch
from torch.profiler import profile, ProfilerActivity
import bench
import paper_2603_25976_b200 as P

dev = torch.device("cuda", 0)
model = P.Model(bench.DIMS[0], bench.DIMS[1:-1], bench.DIMS[-1], "relu")
meth = P.assemble(bench.spec_c3(), model)
w = P.init_params(model, P.Rng(0)).to_device(dev)
hb = bench.make_batches(4, bench.GLOBAL_B, 0, 1)
db = [P.Batch(torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev), "ce", global_size=bench.GLOBAL_B) for X, y in hb]
st = meth.init(w, 0)
for i in range(4):
    w, st, info = meth.step(w, db[i % 4], st)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    w, st, info = meth.step(w, db[0], st)
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
paps = [i for i, e in enumerate(evs) if "k_cg_pap" in e.name]
a, b = paps[3], paps[4]
t0 = evs[a].time_range.end
prev_end = t0
for e in evs[a:b + 1]:
    print(f"{e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f} (+{e.time_range.end - prev_end:6.1f})  {e.name[:70]}")
    prev_end = max(prev_end, e.time_range.end)
