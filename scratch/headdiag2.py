import sys, os; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200._lib as L
if len(sys.argv) > 1: L.LIB_PATH = sys.argv[1]
import paper_2603_25976_b200 as P
from oracle import curvopt_oracle as O
g = np.load("tests/golden/primitives_tc.npz")
name = "relu_ce"
k = lambda s: g[f"{name}/{s}"]
dims = tuple(int(x) for x in k("dims")); act, loss = str(k("act")), str(k("loss"))
m = P.Model(dims[0], dims[1:-1], dims[-1], act)
w = P.ParamVector(k("w"), P.models.param_layout(m))
snap = P.make_snapshot("ggn_ce", m, w, P.Batch(k("X"), k("y"), loss))
lin = O.linearize(dims, act, loss, k("w"), k("X"), k("y"))
ref = O.cg(lambda u: O.ggn_matvec(lin, u), lin.grad, 0.5, 1e-5, 10, 3)
dmv = lambda u: snap.matvec(P.ParamVector(u, w.layout)).data.double().cpu().numpy()
g_dev = snap.grad.data.double().cpu().numpy()
host = O.cg(dmv, g_dev, 0.5, 1e-5, 10, 3)
print("host-driven CG on device products: err %.2e relres %.2e" % (np.linalg.norm(host.x - ref.x) / np.linalg.norm(ref.x), host.relres))
res = P.cg_solve(snap.matvec, snap.grad, 0.5, P.CgConfig(tol=1e-5, maxiter=10, stabilise_every=3))
x = res.direction.data.double().cpu().numpy()
print("device CG: err %.2e relres %.2e" % (np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x), res.final_relative_residual))
# symmetry of the device operator
a, b = O.ORng(1).normal(w.dim), O.ORng(2).normal(w.dim)
print("asym", abs(a @ dmv(b) - b @ dmv(a)) / abs(a @ dmv(b)))
# per-iteration: device CG with maxiter = 1..10
for it in (1, 2, 3, 4, 6, 10):
    r1 = P.cg_solve(snap.matvec, snap.grad, 0.5, P.CgConfig(tol=1e-5, maxiter=it, stabilise_every=3))
    r0 = O.cg(lambda u: O.ggn_matvec(lin, u), lin.grad, 0.5, 1e-5, it, 3)
    print(it, "err %.2e" % (np.linalg.norm(r1.direction.data.double().cpu().numpy() - r0.x) / np.linalg.norm(r0.x)), "relres dev %.3e ref %.3e" % (r1.final_relative_residual, r0.relres))
