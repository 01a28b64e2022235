"""C5 exact-Hessian product at per-rank batches b/N (N = 1, 2, 4, 8): one B200, CUDA events."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2603_25976_b200 as P
dims = bench.WORKLOADS["c5"].dims
model = P.Model(dims[0], dims[1:-1], dims[-1], "relu")
w = P.init_params(model, P.Rng(0)).to_device()
for N in (1, 2, 4, 8):
    b = 32768 // N
    g = np.random.default_rng(N)
    X = torch.from_numpy(g.standard_normal((b, dims[0]), dtype=np.float32)).cuda()
    y = torch.from_numpy(g.integers(0, dims[-1], b)).cuda()
    snap = P.make_snapshot("hessian", model, w, P.Batch(X, y, "ce", global_size=32768))
    v = torch.randn(w.dim, device="cuda"); out = torch.empty_like(v)
    for _ in range(2): snap.apply(1, v, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): snap.apply(1, v, out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    fl = bench.hvp_flops(dims, b)
    print(f"N={N} b={b}: HVP {ms:.2f} ms, {fl / ms / 1e9:.0f} TF/s useful", flush=True)
    snap.close(); del X, y
