"""One C4-size single-GPU row solve and one one-rank distributed solve, each in an NVTX
range (for an ncu launch list filtered by range)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, "/root/repo")
import paper_2603_25976_b200 as P  # noqa: E402
from paper_2603_25976_b200 import _lib  # noqa: E402
from oracle import curvopt_oracle as O  # noqa: E402

dims, b = (3072, 2048, 2048, 10), 4096
m = P.Model(dims[0], dims[1:-1], dims[-1], "relu")
w = P.init_params(m, P.Rng(0))
X, y = O.synthetic_batch(b, dims[0], dims[-1])
snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
mu = float(b)
rt = snap.rt
rhs = snap.row.rhs
lib = _lib.lib()
v1 = snap.row.solve_cholesky(mu)
out = torch.empty_like(v1)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("single")
snap.row.solve_cholesky(mu)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
torch.cuda.nvtx.range_push("dist")
lib.cv_row_solve_cholesky_dist(rt.h, snap.h, C.c_double(mu), C.c_void_p(rhs.data_ptr()), C.c_void_p(out.data_ptr()))
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
