"""Per-iteration vector cost of the device PCG at C3: (solve of n iterations - n products) / n,
CUDA events, tol tiny so every iteration runs; no stabilising iterations."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
from paper_2603_25976_b200.solvers import device_cg, CgConfig
m = P.Model(784, (1024, 1024), 10, "relu")
w = P.init_params(m, P.Rng(0)).to_device()
r = P.Rng(1); b = 8192
X = torch.from_numpy(r.normal(b*784).reshape(b,784).astype(np.float32)).cuda()
y = torch.from_numpy(r.integers(b,10)).cuda()
snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
g = torch.randn(w.dim, device="cuda"); pre = torch.rand(w.dim, device="cuda")
v = torch.randn(w.dim, device="cuda"); out = torch.empty_like(v)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def tprod(n=40):
    for _ in range(3): snap.apply(0, v, out)
    torch.cuda.synchronize(); e0.record()
    for _ in range(n): snap.apply(0, v, out)
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / n
def tsolve(it, reps=10):
    cfg = CgConfig(tol=1e-30, maxiter=it, stabilise_every=0)
    for _ in range(2): device_cg(snap, g, 1.0, cfg, precond=pre)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): device_cg(snap, g, 1.0, cfg, precond=pre)
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / reps
for rep in range(3):
    tp = tprod(); t1 = tsolve(1); t21 = tsolve(21)
    per_it = (t21 - t1) / 20
    print(f"product {tp*1e3:.1f} us; solve(1) {t1*1e3:.1f} us, solve(21) {t21*1e3:.1f} us; per iteration {per_it*1e3:.1f} us "
          f"=> vector part {(per_it - tp)*1e3:.1f} us")
