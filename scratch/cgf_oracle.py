"""k_cg_fused / per-kernel CG iterates against the f64 oracle CG with the device's ReLU masks
(784-512-512-10, b = 256, lam 0.5, no stabilising iteration).  Run with CURVOPT_CG_FUSED=0/1."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
from paper_2603_25976_b200.solvers import device_cg, read_cg_stats, CgConfig
from oracle import curvopt_oracle as O
n0, hid, c = 784, (512, 512), 10
dims = [n0, *hid, c]
m = P.Model(n0, hid, c, "relu")
w = P.init_params(m, P.Rng(3))
r = P.Rng(5); b = 256
Xn = r.normal(b * n0).reshape(b, n0).astype(np.float32); yn = r.integers(b, c)
snap = P.make_snapshot("ggn_ce", m, w.to_device(), P.Batch(torch.from_numpy(Xn).cuda(), torch.from_numpy(yn).cuda(), "ce"))
masks = [(snap.activation(l) > 0).cpu().numpy() for l in range(1, len(dims) - 1)]
lin = O.linearize(dims, "relu", "ce", np.asarray(w.data, dtype=np.float64), Xn, yn, masks=masks)
g = snap.grad.data.clone()
gd = g.double().cpu().numpy()
for it in (3, 5, 7, 9):
    x, st = device_cg(snap, g, 0.5, CgConfig(tol=1e-12, maxiter=it, stabilise_every=0))
    s = read_cg_stats(st)
    o = O.cg(lambda v: O.ggn_matvec(lin, v), gd, 0.5, tol=1e-12, maxiter=it, stabilise_every=0)
    xo = o.x
    xd = x.double().cpu().numpy()
    print(f"maxiter {it}: |x - x_f64|/|x_f64| = {np.linalg.norm(xd - xo) / np.linalg.norm(xo):.2e}  relres dev {s.relres:.5f} f64 {o.relres:.5f}")
