import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
m = P.Model(784, (1024, 1024), 10, "relu")
w = P.init_params(m, P.Rng(0)).to_device()
r = P.Rng(1); b = 8192
X = torch.from_numpy(r.normal(b*784).reshape(b,784).astype(np.float32)).cuda()
y = torch.from_numpy(r.integers(b,10)).cuda()
batch = P.Batch(X, y, "ce")
snap = P.make_snapshot("ggn_ce", m, w, batch)
v = torch.randn(w.dim, device="cuda"); out = torch.empty_like(v)
for _ in range(3): snap.apply(0, v, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): snap.apply(0, v, out)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)/20
print(f"Gv {ms:.3f} ms  {95.7/ms:.1f} TF/s useful")
e0.record()
for _ in range(5):
    s2 = P.make_snapshot("ggn_ce", m, w, batch); s2.close()
e1.record(); torch.cuda.synchronize()
print(f"linearize {e0.elapsed_time(e1)/5:.3f} ms")
