"""C4 lane-equivalence residual ||(G + lam I) d - g|| / ||g|| with the row-lane direction taken
directly from the solve vs recovered from w' - w (fp32 cancellation)."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
b = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
m = P.Model(3072, (2048, 2048), 10, "relu")
w = P.init_params(m, P.Rng(0)).to_device()
r = P.Rng(1); X = torch.from_numpy(r.normal(b*3072).reshape(b,3072).astype(np.float32)).cuda(); y = torch.from_numpy(r.integers(b,10)).cuda()
batch = P.Batch(X, y, "ce")
snap = P.make_snapshot("ggn_ce", m, w, batch)
mu = float(b) * 1.0
v = snap.row.solve_cholesky(mu)
d = snap.row.scaled_row_transpose(v).data
g = snap.grad.data
res = lambda dd: float((snap.matvec(P.ParamVector(dd, w.layout)).data + dd - g).norm() / g.norm())
print(f"b={b} m={b*10}: residual with the solved direction {res(d):.2e}")
meth = P.make("egn_ce", m)
st = meth.init(w, 0)
w1, st, info = meth.step(w, batch, st)
d2 = (w1.data - w.data) / -1e-3
print(f"  with d recovered from (w' - w) / -1e-3 in fp32: {res(d2):.2e} (|u|/|w| = {float((w1.data - w.data).norm() / w.data.norm()):.1e})")
print(f"  rel diff of the two directions {float((d2 - d).norm() / d.norm()):.2e}")
