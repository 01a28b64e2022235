"""Host time between a step's final sync and the next step's graph launch, and the launch's
own host time (C3 graph steps); GPU idle at the step boundary ~ the sum."""
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2603_25976_b200 as P
marks = []
orig_cpu = torch.Tensor.cpu
def cpu(self, *a, **k):
    r = orig_cpu(self, *a, **k)
    marks.append(("sync", time.perf_counter()))
    return r
torch.Tensor.cpu = cpu
orig_replay = torch.cuda.CUDAGraph.replay
def replay(self):
    t0 = time.perf_counter(); orig_replay(self); t1 = time.perf_counter()
    marks.append(("r0", t0)); marks.append(("r1", t1))
torch.cuda.CUDAGraph.replay = replay
dev = torch.device("cuda", 0)
model = P.Model(bench.DIMS[0], bench.DIMS[1:-1], bench.DIMS[-1], "relu")
meth = P.assemble(bench.spec_c3(), model)
w = P.init_params(model, P.Rng(0)).to_device(dev)
hb = bench.make_batches(4, bench.GLOBAL_B, 0, 1)
db = [P.Batch(torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev), "ce", global_size=bench.GLOBAL_B) for X, y in hb]
st = meth.init(w, 0)
for i in range(25):
    w, st, info = meth.step(w, db[i % 4], st)
marks.clear()
for i in range(40):
    w, st, info = meth.step(w, db[i % 4], st)
pre, launch = [], []
last = None
for k, t in marks:
    if k == "sync": last = t
    elif k == "r0" and last is not None: pre.append((t - last) * 1e6); r0 = t
    elif k == "r1" and last is not None: launch.append((t - r0) * 1e6); last = None
print(f"sync -> graph launch call: median {np.median(pre):.0f} us (min {min(pre):.0f}, n={len(pre)})")
print(f"graph launch call (host): median {np.median(launch):.0f} us (min {min(launch):.0f})")
g = next(v for v in meth._graph_cache.values() if v)
try:
    n = g.graph.raw_cuda_graph() if hasattr(g.graph, "raw_cuda_graph") else None
except Exception:
    n = None
print("graph kernels", g.kernels)
