import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
m = P.Model(784, (1024, 1024), 10, "relu")
w = P.init_params(m, P.Rng(0)).to_device()
r = P.Rng(1); b = 8192
X = torch.from_numpy(r.normal(b*784).reshape(b,784).astype(np.float32)).cuda()
y = torch.from_numpy(r.integers(b,10)).cuda()
snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
v = torch.randn(w.dim, device="cuda"); out = torch.empty_like(v)
torch.cuda.synchronize()
print("---- product", file=sys.stderr)
snap.apply(0, v, out)
torch.cuda.synchronize()
