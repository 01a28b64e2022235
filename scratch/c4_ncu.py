"""One C4 planned step inside cudaProfilerStart/Stop (for ncu --profile-from-start off)."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
b = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
m = P.Model(3072, (2048, 2048), 10, "relu")
w = P.init_params(m, P.Rng(0)).to_device()
r = P.Rng(1); X = torch.from_numpy(r.normal(b*3072).reshape(b,3072).astype(np.float32)).cuda(); y = torch.from_numpy(r.integers(b,10)).cuda()
batch = P.Batch(X, y, "ce")
meth = P.make("egn_ce", m); st = meth.init(w, 0)
w1, st, info = meth.step(w, batch, st); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
w1, st, info = meth.step(w, batch, st); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(info)
