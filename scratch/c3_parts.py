"""Composition of a C3 planned step on the device: linearize (snapshot + grad), one GGN
product, the whole PCG solve, the step (eager and graph), by CUDA events."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2603_25976_b200 as P
wl = bench.WORKLOADS["c3"]
dims = wl.dims
model = P.Model(dims[0], dims[1:-1], dims[-1], "relu")
w = P.init_params(model, P.Rng(0)).to_device()
(X, y), = bench.make_batches(1, wl.b, 0, 1, dims)
b = P.Batch(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), "ce")


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


snaps = []
def lin():
    s = P.make_snapshot("ggn_ce", model, w, b)
    snaps.append(s)
    if len(snaps) > 4:
        snaps.pop(0).close()
print(f"linearize (snapshot + loss + grad): {timed(lin):.0f} us")
snap = snaps[-1]
v = torch.randn(w.dim, device="cuda"); out = torch.empty_like(v)
print(f"GGN product: {timed(lambda: snap.apply(0, v, out)):.0f} us")
meth = P.assemble(bench.spec_c3(), model)
st = meth.init(w, 0)
for t in range(12):
    w2, st, info = meth.step(w, b, st)
print("CG iterations per step:", info.solver_iterations)
meth.graphs = False
st2 = meth.init(w, 0)
def step_eager():
    global st2
    _, st2, _ = meth.step(w, b, st2)
print(f"step eager (incl. host sync): {timed(step_eager):.0f} us")
meth.graphs = True
def step_graph():
    global st2
    _, st2, _ = meth.step(w, b, st2)
print(f"step (graphs where eligible): {timed(step_graph):.0f} us")
