import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
b = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
m = P.Model(784, (1024, 1024), 10, "relu")
w = P.init_params(m, P.Rng(0)).to_device()
r = np.random.default_rng(b)
X = torch.from_numpy(r.standard_normal((b, 784), dtype=np.float32)).cuda()
y = torch.from_numpy(r.integers(0, 10, b)).cuda()
snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
v = torch.randn(w.dim, device="cuda"); out = torch.empty_like(v)
for _ in range(3): snap.apply(0, v, out)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
snap.apply(0, v, out); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
