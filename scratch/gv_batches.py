"""GGN product time at the per-rank batch of a dp-N run (b = 8192/N) on one GPU, plus the plans."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
m = P.Model(784, (1024, 1024), 10, "relu")
w = P.init_params(m, P.Rng(0)).to_device()
for b in (8192, 4096, 2048, 1024):
    r = P.Rng(1)
    X = torch.from_numpy(r.normal(b*784).reshape(b,784).astype(np.float32)).cuda()
    y = torch.from_numpy(r.integers(b,10)).cuda()
    snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
    v = torch.randn(w.dim, device="cuda"); out = torch.empty_like(v)
    for _ in range(3): snap.apply(0, v, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): snap.apply(0, v, out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    fl = 8*b*(784*1024+1024*1024+1024*10) - 4*b*784*1024
    print(f"b={b:5d}: Gv {ms*1e3:7.1f} us  {fl/ms/1e9:6.1f} TF/s useful  (x{8192/b:.0f} ranks -> ideal {0.318e3*b/8192:.1f} us)", flush=True)
    snap.close()
