import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
from paper_2603_25976_b200.solvers import _cg_generic
g=np.load('tests/golden/primitives.npz')
n='relu_ce'
dims=tuple(int(x) for x in g[n+'/dims'])
m=P.Model(dims[0],dims[1:-1],dims[-1],'relu')
w=P.ParamVector(g[n+'/w'],P.models.param_layout(m))
snap=P.make_snapshot('ggn_ce',m,w,P.Batch(g[n+'/X'],g[n+'/y'],'ce'))
gg=snap.grad.data
for it in (8,9,10):
    cfg=P.CgConfig(tol=1e-12,maxiter=it,stabilise_every=0)
    x,k,c,rel,_,_=_cg_generic(lambda v: snap.apply(0, v.float().contiguous()), gg.clone(), 0.5, cfg)
    x2,k,c,rel2,_,_=_cg_generic(lambda v: snap.apply(0, v.float().contiguous()).double(), gg.double().clone(), 0.5, cfg)
    r=P.cg_solve(snap.matvec,snap.grad,0.5,cfg)
    print(it, 'torch-f32', rel, 'torch-f64vec', rel2, 'native', r.final_relative_residual)
