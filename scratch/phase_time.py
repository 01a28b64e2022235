"""Per-phase device time of C3 planned steps: linearize (make_snapshot), solve, rest (CUDA events)."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import gc, os
if os.environ.get("NO_GC"): gc.disable()
import bench
import paper_2603_25976_b200 as P
import paper_2603_25976_b200.method as M

dev = torch.device("cuda", 0)
model = P.Model(bench.DIMS[0], bench.DIMS[1:-1], bench.DIMS[-1], "relu")
meth = P.assemble(bench.spec_c3(), model)
w = P.init_params(model, P.Rng(0)).to_device(dev)
hb = bench.make_batches(4, bench.GLOBAL_B, 0, 1)
db = [P.Batch(torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev), "ce", global_size=bench.GLOBAL_B) for X, y in hb]
st = meth.init(w, 0)
ev = []
orig_mk = M.make_snapshot
orig_solve = meth._solve
def mk(*a, **k):
    e0 = torch.cuda.Event(enable_timing=True); e0.record(); s = orig_mk(*a, **k)
    e1 = torch.cuda.Event(enable_timing=True); e1.record(); ev.append(("lin", e0, e1)); return s
def solve(*a, **k):
    e0 = torch.cuda.Event(enable_timing=True); e0.record(); r = orig_solve(*a, **k)
    e1 = torch.cuda.Event(enable_timing=True); e1.record(); ev.append(("solve", e0, e1)); return r
M.make_snapshot = mk
meth._solve = solve
for i in range(5):
    w, st, info = meth.step(w, db[i % 4], st)
torch.cuda.synchronize(); ev.clear()
N = 20
s0 = torch.cuda.Event(enable_timing=True); s0.record()
prods = 0
for i in range(N):
    w, st, info = meth.step(w, db[i % 4], st)
    prods += meth.last_products
s1 = torch.cuda.Event(enable_timing=True); s1.record(); torch.cuda.synchronize()
tot = s0.elapsed_time(s1) / N
agg = {}
for k, a, b in ev: agg[k] = agg.get(k, 0.0) + a.elapsed_time(b) / N
print(f"step {tot:.3f} ms; products/step {prods / N:.1f}; " + ", ".join(f"{k} {v:.3f} ms" for k, v in agg.items()) +
      f"; rest {tot - sum(agg.values()):.3f} ms")
