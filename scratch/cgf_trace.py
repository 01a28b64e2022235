"""Per-block timeline of k_cg_fused (globaltimer stamps per phase).  Needs a temporary
instrumentation patch of csrc/vec.cu that is NOT in the tree: a `trace` pointer in
CgFusedArgs read from CURVOPT_CGF_TRACE (a device address) and TR(k) stamps at kernel
entry, barrier arrivals/releases and exit (results: profiles/r3_cg_fused.txt)."""
import sys, os; sys.path.insert(0, ".")
import numpy as np, torch
buf = torch.zeros(592 * 8, dtype=torch.int64, device="cuda")
os.environ["CURVOPT_CGF_TRACE"] = str(buf.data_ptr())
import paper_2603_25976_b200 as P
from paper_2603_25976_b200.solvers import device_cg, CgConfig
m = P.Model(784, (1024, 1024), 10, "relu")
w = P.init_params(m, P.Rng(0)).to_device()
r = P.Rng(1); b = 8192
X = torch.from_numpy(r.normal(b*784).reshape(b,784).astype(np.float32)).cuda()
y = torch.from_numpy(r.integers(b,10)).cuda()
snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
g = torch.randn(w.dim, device="cuda"); pre = torch.rand(w.dim, device="cuda")
for it in (1, 2, 3):
    buf.zero_()
    device_cg(snap, g, 1.0, CgConfig(tol=1e-30, maxiter=it, stabilise_every=0), precond=pre)
    torch.cuda.synchronize()
    t = buf.view(592, 8).cpu().numpy().astype(np.float64)
    t0 = t[:, 0].min()
    t = (t - t0) / 1e3
    names = ["entry", "arrive1", "decided1", "arrive2", "after2dec", "end", "released1", "released2"]
    for k, n in enumerate(names):
        col = t[:, k]; col = col[col > -1e6]
        nz = col[col >= 0]
        if len(nz): print(f"  {n:10s} min {nz.min():7.2f} med {np.median(nz):7.2f} max {nz.max():7.2f} us")
    print("--")
