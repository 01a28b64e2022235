import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
from oracle import curvopt_oracle as O
g=np.load('tests/golden/primitives.npz')
def rel(a,b):
    a=a.detach().double().cpu().numpy() if hasattr(a,'detach') else np.asarray(a); b=np.asarray(b)
    return np.linalg.norm(a.ravel()-b.ravel())/np.linalg.norm(b.ravel())
for n in ['relu_ce','tanh_ce','relu_mse','tanh_mse','lin_ce']:
    k=lambda s: g[n+'/'+s]
    dims=tuple(int(x) for x in k('dims'))
    m=P.Model(dims[0],dims[1:-1],dims[-1],str(k('act')))
    w=P.ParamVector(k('w'),P.models.param_layout(m))
    loss=str(k('loss'))
    snap=P.make_snapshot('ggn_ce' if loss=='ce' else 'ggn_mse',m,w,P.Batch(k('X'),k('y'),loss))
    v=P.ParamVector(k('v'),w.layout)
    print(n, 'grad %.2e jvp %.2e vjp %.2e ggn %.2e hvp %.2e out %.2e' % (rel(snap.grad.data,k('grad')), rel(snap.jvp(v),k('jvp')), rel(snap.vjp(k('U')).data,k('vjp')), rel(snap.matvec(v).data,k('ggn')), rel(snap.hvp(v).data,k('hvp')), rel(snap.outputs(),k('out'))))
    lin=O.linearize(dims,str(k('act')),loss,k('w'),k('X'),k('y'))
    p=snap.grad.data.clone()
    ref=O.ggn_matvec(lin,p.double().cpu().numpy())
    print('   ggn(g) %.2e' % rel(snap.matvec(P.ParamVector(p,w.layout)).data, ref))
