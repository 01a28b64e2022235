import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
from paper_2603_25976_b200.runtime import runtime
from oracle import curvopt_oracle as O
rt = runtime()
def rel(a,b): a=a.double().cpu(); b=b.double().cpu(); return float((a-b).norm()/b.norm())
for dims,b,act,loss in [((3072,512,512,10),96,'tanh','ce'),((784,1024,1024,10),256,'tanh','ce'),((3072,512,512,10),512,'tanh','ce')]:
    m=P.Model(dims[0],dims[1:-1],dims[-1],act); w=P.init_params(m,P.Rng(0)); r=P.Rng(1)
    X=r.normal(b*dims[0]).reshape(b,dims[0]); y=r.integers(b,dims[-1])
    batch=P.Batch(X,y,loss); vv=P.Rng(2).normal(w.dim); v=P.ParamVector(vv,w.layout)
    lin=O.linearize(dims,act,loss,w.data,X,y)
    ref=dict(g=lin.grad, gv=O.ggn_matvec(lin,vv), hv=O.hvp(lin,vv))
    for eng in ('simt','auto'):
        rt.set_engine(eng); s=P.make_snapshot('ggn_ce',m,w,batch)
        got=dict(g=s.grad.data, gv=s.matvec(v).data, hv=s.hvp(v).data)
        print(dims,b,eng, {k: '%.2e'%rel(got[k], torch.tensor(ref[k])) for k in ref})
        s.close()
rt.set_engine('auto')
