import sys; sys.path.insert(0, ".")
import numpy as np, torch, time
import paper_2603_25976_b200 as P
from paper_2603_25976_b200.runtime import runtime
from oracle import curvopt_oracle as O
dims=(784,1024,1024,10); b=int(sys.argv[1]) if len(sys.argv)>1 else 8192
m=P.Model(784,(1024,1024),10,'relu'); w=P.init_params(m,P.Rng(0))
X,y=O.synthetic_batch(b,784,10)
spec=P.MethodSpec(curvature=P.CurvatureSpec('ggn_ce'), solver=P.SolverSpec('cg',P.CgConfig(tol=1e-5,maxiter=10,stabilise_every=10)),
   damping=P.DampingSpec('constant',1.0), chain=(P.transforms.scale(1e-3),P.transforms.scale(-1.0)))
for eng in ('simt','auto'):
    runtime().set_engine(eng)
    meth=P.assemble(spec,m); st=meth.init(w,0)
    snap=P.make_snapshot('ggn_ce',m,w,P.Batch(X,y,'ce'))
    masks=[(snap.activation(l)>0).cpu().numpy() for l in (1,2)]; snap.close()
    w1,st,info=meth.step(w,P.Batch(X,y,'ce'),st)
    d=st.warm_start.double().cpu().numpy()
    t=time.time()
    os_=O.OSpec(); ost=O.oracle_init(os_,w.dim)
    _,_,oinfo,odir=O.oracle_step(os_,dims,'relu','ce',w.data,X,y,ost,masks=masks)
    print(eng, 'iters', info.solver_iterations, oinfo['solver_iterations'], 'relres', info.final_relative_residual, oinfo['final_relative_residual'],
          'dir rel err %.2e' % (np.linalg.norm(d-odir)/np.linalg.norm(odir)), 'loss rel %.1e' % abs(info.loss_before/oinfo['loss_before']-1), 'oracle %.1fs'%(time.time()-t))
