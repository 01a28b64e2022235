"""Host-side timing of Method.step phases (C3) to locate GPU idle gaps."""
import sys, time, collections
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2603_25976_b200 as P
import paper_2603_25976_b200.method as M

T = collections.defaultdict(float)
def wrap(mod, name):
    f = getattr(mod, name)
    def g(*a, **k):
        t0 = time.perf_counter(); r = f(*a, **k); T[name] += time.perf_counter() - t0; return r
    setattr(mod, name, g)
wrap(M, "make_snapshot")
orig_pc = M.Method._solve_param_cg
def solve(self, *a, **k):
    t0 = time.perf_counter(); r = orig_pc(self, *a, **k); T["_solve"] += time.perf_counter() - t0; return r
M.Method._solve_param_cg = solve
orig_cpu = torch.Tensor.cpu
def cpu(self, *a, **k):
    t0 = time.perf_counter(); r = orig_cpu(self, *a, **k); T["cpu(sync)"] += time.perf_counter() - t0; return r
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
torch.cuda.synchronize()
T.clear()
N = 20
t0 = time.perf_counter()
for i in range(N):
    w, st, info = meth.step(w, db[i % 4], st)
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / N
print(f"step wall {tot*1e3:.3f} ms")
for k, v in T.items():
    print(f"  {k:14s} {v/N*1e3:.3f} ms")
