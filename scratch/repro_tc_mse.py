import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_25976_b200 as P
from oracle import curvopt_oracle as O
dims = tuple(int(x) for x in sys.argv[1].split(","))
b = int(sys.argv[2]); act = sys.argv[3]; loss = sys.argv[4]
m = P.Model(dims[0], dims[1:-1], dims[-1], act)
w = P.init_params(m, P.Rng(0))
X, y = O.synthetic_batch(b, dims[0], dims[-1], loss=loss)
snap = P.make_snapshot("ggn_ce" if loss == "ce" else "ggn_mse", m, w, P.Batch(X, y, loss))
torch.cuda.synchronize(); print("linearize ok", flush=True)
v = P.ParamVector(O.ORng(2).normal(w.dim), w.layout)
out = snap.jvp(v); torch.cuda.synchronize(); print("jvp ok", flush=True)
g = snap.matvec(v); torch.cuda.synchronize(); print("ggn ok", flush=True)
h = snap.hvp(v); torch.cuda.synchronize(); print("hvp ok", flush=True)
