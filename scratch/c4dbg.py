import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
from paper_2603_25976_b200.runtime import runtime
from oracle import curvopt_oracle as O
b = int(sys.argv[1]); dims=(int(sys.argv[2]),)+tuple(int(x) for x in sys.argv[3].split(','))+(10,)
m = P.Model(dims[0], dims[1:-1], 10, "relu")
w = P.init_params(m, P.Rng(0))
X, y = O.synthetic_batch(b, dims[0], 10)
for eng in ("simt", "auto"):
    runtime().set_engine(eng)
    snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
    masks=[(snap.activation(l)>0).cpu().numpy() for l in range(1, len(dims)-1)]
    lin = O.linearize(dims,'relu','ce',w.data,X,y,masks=masks)
    seeds, rhs = O.row_seeds_rhs(lin)
    G = O.output_gram(lin, seeds)
    Gd = snap.row.gram().double().cpu().numpy()
    rd = snap.row.rhs.double().cpu().numpy()
    mu = float(b)
    v = O.row_cholesky(G, rhs, mu)
    vd = snap.row.solve_cholesky(mu).double().cpu().numpy()
    vdd = np.linalg.solve(Gd + mu*np.eye(len(rd)), rd)   # exact solve of the DEVICE system
    d_o = O.row_transpose(lin, seeds, v)
    d_d = snap.row.scaled_row_transpose(torch.tensor(vd, dtype=torch.float32)).data.double().cpu().numpy()
    e = lambda a, r: np.linalg.norm(a - r) / np.linalg.norm(r)
    print(eng, "gram %.2e rhs %.2e | v(chol dev) vs v(oracle) %.2e | v(exact dev sys) vs oracle %.2e | chol vs exact-dev %.2e | dir %.2e  cond~%.1e" % (
        e(Gd, G), e(rd, rhs), e(vd, v), e(vdd, v), e(vd, vdd), e(d_d, d_o), np.linalg.cond(G + mu*np.eye(len(rhs)))))
    snap.close()
