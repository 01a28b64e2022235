"""Find the first native call that invalidates a step capture."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from cuda.bindings import runtime as cr
import paper_2603_25976_b200 as P
from paper_2603_25976_b200.runtime import runtime
from oracle import curvopt_oracle as O
rt = runtime()
orig = rt.call
def status():
    s = torch.cuda.current_stream().cuda_stream
    r = cr.cudaStreamGetCaptureInfo(s)
    return r[1]
def traced(name, *args):
    before = status()
    orig(name, *args)
    after = status()
    print(f"{name}: {before} -> {after}", flush=True)
rt.call = traced
model = P.Model(784, (256, 128), 10, "relu")
X, y = O.synthetic_batch(512, 784, 10, seed=1)
Xd, yd = torch.from_numpy(X.astype(np.float32)).cuda(), torch.from_numpy(y).cuda()
cg = P.CgConfig(tol=1e-5, maxiter=6, stabilise_every=4, warm_start=True)
spec = P.MethodSpec(curvature=P.CurvatureSpec("ggn_ce"), solver=P.SolverSpec("cg", cg),
                    damping=P.DampingSpec("constant", 1.0), chain=(P.transforms.scale(1e-3), P.transforms.scale(-1.0)))
meth = P.assemble(spec, model)
w = P.init_params(model, P.Rng(0)).to_device()
st = meth.init(w, 0)
for i in range(3):
    print("---- step", i, flush=True)
    try:
        w, st, info = meth.step(w, P.Batch(Xd, yd, "ce"), st)
    except Exception as e:
        import traceback
        print("EXC", type(e).__name__, str(e)[:200])
        c = e.__context__
        while c is not None:
            print("CONTEXT:", type(c).__name__, str(c)[:500])
            traceback.print_tb(c.__traceback__)
            c = c.__context__
        break
