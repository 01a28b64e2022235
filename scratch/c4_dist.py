"""C4 (3072-2048-2048-10 CE, b=4096, m=40,960) row solve: single-GPU path vs the
distributed row lane on one rank, and the per-rank compute of the distributed lane at
world = 2/4/8 (a context of that world size with no communicator: each 'rank' does its
own share of the SYRK strips, panel factorizations and trailing updates; collectives are
skipped, so results are garbage and only the timing is meaningful)."""
import ctypes as C
import sys
import time

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


def timed(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return min(ts)


v1 = snap.row.solve_cholesky(mu)
print(f"single-GPU solve_cholesky (Gram cached after the first call): {timed(lambda: snap.row.solve_cholesky(mu)):.1f} ms")
out = torch.empty_like(v1)


def dist(ctx):
    rc = lib.cv_row_solve_cholesky_dist(ctx, snap.h, C.c_double(mu), C.c_void_p(rhs.data_ptr()),
                                        C.c_void_p(out.data_ptr()))
    return rc


print(f"distributed lane, one rank (Gram strips rebuilt each call): {timed(lambda: dist(rt.h)):.1f} ms")
e = float((out.double() - v1.double()).norm() / v1.double().norm())
print(f"  vs single-GPU solve: {e:.2e}")
for W in (2, 4, 8):
    ts = []
    for r in range(W):
        h = C.c_void_p()
        assert lib.cv_ctx_create(0, W, r, None, C.byref(h)) == 0
        lib.cv_ctx_set_stream(h, C.c_void_p(torch.cuda.current_stream().cuda_stream))
        ts.append(timed(lambda: dist(h), reps=2))
        lib.cv_ctx_destroy(h)
    print(f"world {W}: per-rank compute (no communication) max {max(ts):.1f} ms, min {min(ts):.1f} ms "
          f"(factor + solves; ranks whose factor hits a garbage pivot skip the solves)")
