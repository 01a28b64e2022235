"""Host time between a step's final sync and the next step's first native call (GPU idle)."""
import sys, time; sys.path.insert(0, ".")
import torch
import bench
import paper_2603_25976_b200 as P
import paper_2603_25976_b200.method as M
from paper_2603_25976_b200 import _lib
marks = []
orig_mk = M.make_snapshot
def mk(*a, **k):
    marks.append(("mk", time.perf_counter()))
    return orig_mk(*a, **k)
M.make_snapshot = mk
orig_cpu = torch.Tensor.cpu
def cpu(self, *a, **k):
    r = orig_cpu(self, *a, **k)
    marks.append(("sync", time.perf_counter()))
    return r
torch.Tensor.cpu = cpu
dev = torch.device("cuda", 0)
model = P.Model(bench.DIMS[0], bench.DIMS[1:-1], bench.DIMS[-1], "relu")
meth = P.assemble(bench.spec_c3(), model)
w = P.init_params(model, P.Rng(0)).to_device(dev)
hb = bench.make_batches(4, bench.GLOBAL_B, 0, 1)
db = [P.Batch(torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev), "ce", global_size=bench.GLOBAL_B) for X, y in hb]
st = meth.init(w, 0)
for i in range(5):
    w, st, info = meth.step(w, db[i % 4], st)
marks.clear()
for i in range(30):
    w, st, info = meth.step(w, db[i % 4], st)
gaps = []
last_sync = None
for kind, t in marks:
    if kind == "sync":
        last_sync = t
    elif kind == "mk" and last_sync is not None:
        gaps.append((t - last_sync) * 1e6)
        last_sync = None
gaps.sort()
print(f"sync -> next make_snapshot: median {gaps[len(gaps)//2]:.0f} us, min {gaps[0]:.0f}, max {gaps[-1]:.0f} (n={len(gaps)})")
