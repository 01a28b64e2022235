import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
g=np.load('tests/golden/primitives.npz')
n='relu_ce'
dims=tuple(int(x) for x in g[n+'/dims'])
m=P.Model(dims[0],dims[1:-1],dims[-1],'relu')
w=P.ParamVector(g[n+'/w'],P.models.param_layout(m))
snap=P.make_snapshot('ggn_ce',m,w,P.Batch(g[n+'/X'],g[n+'/y'],'ce'))
for stab in (3, 0):
  for it in range(1,11):
    r=P.cg_solve(snap.matvec,snap.grad,0.5,P.CgConfig(tol=1e-12,maxiter=it,stabilise_every=stab))
    print(stab, it, r.iterations, r.relres if hasattr(r,'relres') else r.final_relative_residual, r.gv_count)
