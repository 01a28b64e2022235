"""GGN product time at per-rank batches: eager launches vs one CUDA-graph replay."""
import sys, ctypes as C; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
from paper_2603_25976_b200.runtime import runtime
rt = runtime()
dims = (784, 1024, 1024, 10)
m = P.Model(784, (1024, 1024), 10, "relu")
w = P.init_params(m, P.Rng(0)).to_device()
for b in (256, 1024, 2048, 8192):
    r = np.random.default_rng(b)
    X = torch.from_numpy(r.standard_normal((b, 784), dtype=np.float32)).cuda()
    y = torch.from_numpy(r.integers(0, 10, b)).cuda()
    snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
    v = torch.randn(w.dim, device="cuda"); out = torch.empty_like(v)
    for _ in range(3): snap.apply(0, v, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): snap.apply(0, v, out)
    e1.record(); torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) / 20
    n0 = rt.launches()
    g = torch.cuda.CUDAGraph()
    rt.lib.cv_ctx_capture_begin(rt.h)
    arena = C.c_void_p()
    with torch.cuda.graph(g, capture_error_mode="relaxed"):
        rt.bind_stream()
        for _ in range(5): snap.apply(0, v, out)
    rt.lib.cv_ctx_capture_end(rt.h, C.byref(arena)); rt.bind_stream()
    k = (rt.launches() - n0) / 5
    g.replay(); torch.cuda.synchronize()
    e0.record()
    for _ in range(4): g.replay()
    e1.record(); torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / 20
    gf = (8 * b * (784 * 1024 + 1024 * 1024 + 1024 * 10) - 4 * b * 784 * 1024) / 1e9
    print(f"b={b}: eager {eager * 1e3:.1f} us, graph {graph * 1e3:.1f} us, {k:.0f} kernels/product, "
          f"{gf:.1f} GF -> {gf / graph:.0f} TF/s (graph)")
    del g; snap.close()
