"""Fused vs per-kernel CG iterates for increasing maxiter (run with CURVOPT_CG_FUSED=0/1, writes npz)."""
import sys, os; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
from paper_2603_25976_b200.solvers import device_cg, read_cg_stats, CgConfig
res = {}
for n0, hid, c in [(784, (256, 256), 10), (784, (512, 512), 10), (784, (1024, 1024), 10)]:
    m = P.Model(n0, hid, c, "relu")
    w = P.init_params(m, P.Rng(3)).to_device()
    r = P.Rng(5); b = 256
    X = torch.from_numpy(r.normal(b * n0).reshape(b, n0).astype(np.float32)).cuda()
    batch = P.Batch(X, torch.from_numpy(r.integers(b, c)).cuda(), "ce")
    snap = P.make_snapshot("ggn_ce", m, w, batch)
    g = snap.grad.data.clone()
    for it in (1, 2, 3, 5, 9):
        x, st = device_cg(snap, g, 0.5, CgConfig(tol=1e-12, maxiter=it, stabilise_every=0))
        s = read_cg_stats(st)
        res[f"{w.dim}_{it}"] = x.double().cpu().numpy()
        res[f"{w.dim}_{it}_rr"] = np.array([s.relres, s.iterations])
np.savez(sys.argv[1], **res)
