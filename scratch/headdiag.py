import sys, os; sys.path.insert(0, ".")
import numpy as np
import paper_2603_25976_b200._lib as L
if len(sys.argv) > 1: L.LIB_PATH = sys.argv[1]
import paper_2603_25976_b200 as P
from oracle import curvopt_oracle as O
g = np.load("tests/golden/primitives_tc.npz")
for name in ("relu_ce", "tanh_ce", "relu_mse"):
    k = lambda s: g[f"{name}/{s}"]
    dims = tuple(int(x) for x in k("dims")); act, loss = str(k("act")), str(k("loss"))
    m = P.Model(dims[0], dims[1:-1], dims[-1], act)
    w = P.ParamVector(k("w"), P.models.param_layout(m))
    snap = P.make_snapshot("ggn_ce" if loss == "ce" else "ggn_mse", m, w, P.Batch(k("X"), k("y"), loss))
    lin = O.linearize(dims, act, loss, k("w"), k("X"), k("y"))
    errs = []
    for i in range(4):
        v = O.ORng(10 + i).normal(w.dim)
        d = snap.matvec(P.ParamVector(v, w.layout)).data.double().cpu().numpy()
        o = O.ggn_matvec(lin, v)
        errs.append(np.linalg.norm(d - o) / np.linalg.norm(o))
    res = P.cg_solve(snap.matvec, snap.grad, 0.5, P.CgConfig(tol=1e-5, maxiter=10, stabilise_every=3))
    ref = O.cg(lambda u: O.ggn_matvec(lin, u), lin.grad, 0.5, 1e-5, 10, 3)
    e = np.linalg.norm(res.direction.data.double().cpu().numpy() - ref.x) / np.linalg.norm(ref.x)
    print(name, "product errs", ["%.1e" % x for x in errs], "cg err %.2e relres dev %.2e ref %.2e" % (e, res.final_relative_residual, ref.relres))
