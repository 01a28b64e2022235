import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
which = sys.argv[1]; b = int(sys.argv[2])
def tsync(): torch.cuda.synchronize(); return time.time()
if which == "c4":
    m = P.Model(3072, (2048, 2048), 10, "relu")
    w = P.init_params(m, P.Rng(0)).to_device()
    r = P.Rng(1); X = torch.from_numpy(r.normal(b*3072).reshape(b,3072).astype(np.float32)).cuda(); y = torch.from_numpy(r.integers(b,10)).cuda()
    batch = P.Batch(X, y, "ce")
    meth = P.make("egn_ce", m)   # ggn_ce + row_cholesky, lam 1
    st = meth.init(w, 0)
    t0 = tsync(); w1, st, info = meth.step(w, batch, st); t1 = tsync()
    print("C4 step", b, "m", b*10, "time %.3f s" % (t1-t0), info.loss_before, info.step_norm)
    t0 = tsync(); w1, st, info = meth.step(w, batch, st); t1 = tsync()
    print("C4 step (warm)", "time %.3f s" % (t1-t0))
    # property: the row-lane direction solves (G + lam I) d = g   (lane equivalence)
    snap = P.make_snapshot("ggn_ce", m, w, batch)
    d = (w1.data - w.data) / -1e-3
    gd = snap.matvec(P.ParamVector(d, w.layout)).data + 1.0 * d
    res = float((gd - snap.grad.data).norm() / snap.grad.data.norm())
    print("C4 lane-equivalence residual ||(G+lam I)d - g||/||g|| = %.2e" % res)
else:
    m = P.Model(3072, (4096,)*4, 10, "relu")
    w = P.init_params(m, P.Rng(0)).to_device()
    r = P.Rng(1); X = torch.from_numpy(r.normal(b*3072).reshape(b,3072).astype(np.float32)).cuda(); y = torch.from_numpy(r.integers(b,10)).cuda()
    batch = P.Batch(X, y, "ce")
    spec = P.MethodSpec(curvature=P.CurvatureSpec("hessian"), solver=P.SolverSpec("cg", P.CgConfig(tol=1e-5, maxiter=10, stabilise_every=10)),
                        damping=P.DampingSpec("constant", 1.0), estimator=P.EstimatorSpec("hutchinson", 1, every_k=10),
                        telemetry=P.TelemetrySpec(trace_every_k=10), chain=(P.transforms.scale(1e-3), P.transforms.scale(-1.0)))
    meth = P.assemble(spec, m); st = meth.init(w, 0)
    for i in range(3):
        t0 = tsync(); w, st, info = meth.step(w, batch, st); t1 = tsync()
        print("C5 step", i, b, "time %.3f s" % (t1-t0), "iters", info.solver_iterations, "trace", info.trace_estimate, "diag_mean", info.diag_mean, "products", meth.last_products)
    snap = P.make_snapshot("hessian", m, w, batch)
    v = torch.randn(w.dim, device="cuda"); out = torch.empty_like(v)
    snap.apply(1, v, out); t0 = tsync()
    for _ in range(3): snap.apply(1, v, out)
    t1 = tsync(); hv = (t1-t0)/3
    L = [3072]+[4096]*4+[10]; Pw = sum(L[i]*L[i+1] for i in range(5)); fl = 12*b*Pw - 8*b*L[0]*L[1]
    print("C5 HVP %.3f ms  %.1f TF/s useful" % (hv*1e3, fl/hv/1e12))
if which == "c4o":
    from oracle import curvopt_oracle as O
    dims=(3072,2048,2048,10)
    m = P.Model(3072, (2048, 2048), 10, "relu")
    w = P.init_params(m, P.Rng(0))
    X, y = O.synthetic_batch(b, 3072, 10)
    meth = P.make("egn_ce", m); st = meth.init(w, 0)
    snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
    masks=[(snap.activation(l)>0).cpu().numpy() for l in (1,2)]; snap.close()
    w1, st, info = meth.step(w, P.Batch(X, y, "ce"), st)
    d = (w1.data - w.data) / -1e-3
    t=time.time()
    os_=O.OSpec(solver="row_cholesky"); ost=O.oracle_init(os_, w.dim)
    _,_,oinfo,odir=O.oracle_step(os_,dims,'relu','ce',w.data,X,y,ost,masks=masks)
    print("C4 b=%d dir rel err %.2e (oracle %.1fs)" % (b, np.linalg.norm(d-odir)/np.linalg.norm(odir), time.time()-t))
