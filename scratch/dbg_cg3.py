import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
from paper_2603_25976_b200.solvers import _cg_generic
from oracle import curvopt_oracle as O
g=np.load('tests/golden/primitives.npz')
n='relu_ce'
dims=tuple(int(x) for x in g[n+'/dims'])
m=P.Model(dims[0],dims[1:-1],dims[-1],'relu')
w=P.ParamVector(g[n+'/w'],P.models.param_layout(m))
snap=P.make_snapshot('ggn_ce',m,w,P.Batch(g[n+'/X'],g[n+'/y'],'ce'))
lin=O.linearize(dims,'relu','ce',g[n+'/w'],g[n+'/X'],g[n+'/y'])
gg=snap.grad.data
for it in range(1,11):
    cfg=P.CgConfig(tol=1e-12,maxiter=it,stabilise_every=0)
    x,k,c,rel,_,_=_cg_generic(lambda v: snap.apply(0, v.float().contiguous()), gg.clone(), 0.5, cfg)
    r=P.cg_solve(snap.matvec,snap.grad,0.5,cfg)
    xn=r.direction.data
    ref=O.cg(lambda v:O.ggn_matvec(lin,v), lin.grad, 0.5, 1e-12, it, 0).x
    e=lambda a: np.linalg.norm(a.double().cpu().numpy()-ref)/np.linalg.norm(ref)
    # true residual of each
    def tr(xx):
        xx=xx.double().cpu().numpy(); rr=lin.grad-(O.ggn_matvec(lin,xx)+0.5*xx); return np.linalg.norm(rr)/np.linalg.norm(lin.grad)
    print(it, 'torch err %.2e true %.3e rec %.3e | native err %.2e true %.3e rec %.3e' % (e(x), tr(x), rel, e(xn), tr(xn), r.final_relative_residual))
