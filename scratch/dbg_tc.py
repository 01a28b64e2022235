import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2603_25976_b200.runtime import runtime
rt = runtime()
M=N=128; K=32
for a_km, b_km in ((1,1),(0,1),(1,0)):
    A = (torch.arange(M, device='cuda').float()[:,None]*1 + torch.arange(K, device='cuda').float()[None,:]*1000)
    B = torch.eye(K, N, device='cuda')
    a = A.contiguous() if a_km else A.t().contiguous()
    b = B.t().contiguous() if b_km else B.contiguous()
    lda = K if a_km else M; ldb = K if b_km else N
    stage = 2*M*K + 2*N*K
    out = torch.zeros(M*N + stage, device='cuda')
    rt.call("cv_gemm_test", rt.h, 3, M, N, K, a.data_ptr(), lda, a_km, b.data_ptr(), ldb, b_km, out.data_ptr(), N)
    torch.cuda.synchronize()
    C = out[:M*N].view(M,N); S = out[M*N:].cpu().numpy()
    ref = A @ B
    print('case a_km', a_km, 'b_km', b_km, 'err', float((C-ref).norm()/ref.norm()))
    Ahi = S[:M*K]; Bhi = S[2*M*K:2*M*K+N*K]
    print(' A smem first 40:', Ahi[:40].astype(int).tolist())
    print(' A smem @1024 floats (4KB):', Ahi[1024:1032].astype(int).tolist(), 'nonzero count', int((Ahi!=0).sum()))
    print(' B smem nonzero', int((Bhi!=0).sum()), 'first nz idx', np.nonzero(Bhi)[0][:10].tolist())
    print(' C[0:3,0:6]', C[:3,:6].cpu().numpy().tolist())
