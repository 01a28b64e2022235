"""C5 planned steps (b=32768, 3072-4096x4-10, HVP + CG + Hutchinson/trace @10); step 10 (estimator
and trace fire) inside cudaProfilerStart/Stop."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2603_25976_b200 as P
wl = bench.WORKLOADS["c5"]
dims = wl.dims
model = P.Model(dims[0], dims[1:-1], dims[-1], "relu")
meth = P.assemble(bench.spec_c5(), model)
meth.graphs = False
w = P.init_params(model, P.Rng(0)).to_device()
(X, y), = bench.make_batches_fast(1, wl.b, 0, 1, dims)
b = P.Batch(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), "ce")
st = meth.init(w, 0)
for t in range(10):
    w, st, info = meth.step(w, b, st)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
w, st, info = meth.step(w, b, st)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(info)
