"""Which host call stalls in the second estimator step (t=10)?"""
import sys, time; sys.path.insert(0, ".")
import torch
import bench
import paper_2603_25976_b200 as P
import paper_2603_25976_b200.method as M
from paper_2603_25976_b200.runtime import Runtime
T = {}
def timed(obj, name, label):
    f = getattr(obj, name)
    def g(*a, **k):
        t0 = time.perf_counter(); r = f(*a, **k); T[label] = T.get(label, 0.0) + time.perf_counter() - t0; return r
    setattr(obj, name, g)
timed(M, "make_snapshot", "make_snapshot")
timed(M, "device_hutchinson", "hutchinson")
orig_call = Runtime.call
def call(self, name, *a):
    t0 = time.perf_counter(); r = orig_call(self, name, *a); T["call:" + name] = T.get("call:" + name, 0.0) + time.perf_counter() - t0; return r
Runtime.call = call
orig_clone = torch.Tensor.clone
def clone(self, *a, **k):
    t0 = time.perf_counter(); r = orig_clone(self, *a, **k); T["clone"] = T.get("clone", 0.0) + time.perf_counter() - t0; return r
torch.Tensor.clone = clone
dev = torch.device("cuda", 0)
model = P.Model(bench.DIMS[0], bench.DIMS[1:-1], bench.DIMS[-1], "relu")
meth = P.assemble(bench.spec_c3(), model)
w = P.init_params(model, P.Rng(0)).to_device(dev)
hb = bench.make_batches(4, bench.GLOBAL_B, 0, 1)
db = [P.Batch(torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev), "ce", global_size=bench.GLOBAL_B) for X, y in hb]
st = meth.init(w, 0)
for i in range(22):
    T.clear()
    a0 = torch.cuda.memory_stats().get("num_device_alloc", 0)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    w, st, info = meth.step(w, db[i % 4], st)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    a1 = torch.cuda.memory_stats().get("num_device_alloc", 0)
    if i in (0, 1, 10, 11, 20):
        top = sorted(T.items(), key=lambda kv: -kv[1])[:5]
        print(i, f"{dt*1e3:.2f} ms torch_dev_allocs+{a1-a0}", [(k, round(v * 1e3, 2)) for k, v in top])
