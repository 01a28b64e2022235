"""One C5 exact-Hessian product (b=32768, 3072-4096x4-10) inside cudaProfilerStart/Stop,
after a warm one (for ncu --profile-from-start off --set full)."""
import sys; sys.path.insert(0, ".")
import torch
import bench
import paper_2603_25976_b200 as P
wl = bench.WORKLOADS["c5"]
dims = wl.dims
model = P.Model(dims[0], dims[1:-1], dims[-1], "relu")
w = P.init_params(model, P.Rng(0)).to_device()
(X, y), = bench.make_batches_fast(1, wl.b, 0, 1, dims)
b = P.Batch(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), "ce")
snap = P.make_snapshot("hessian", model, w, b)
v = torch.randn(w.dim, device="cuda")
out = torch.empty_like(v)
snap.apply(1, v, out)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
snap.apply(1, v, out)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
