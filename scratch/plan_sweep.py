"""Time GEMM shapes of small-batch products under forced tile kinds / split-K factors."""
import sys, ctypes as C; sys.path.insert(0, ".")
import torch
from paper_2603_25976_b200.runtime import runtime
rt = runtime()
ms = C.c_float()
def t(M, N, K, ak, bk, mode, kind, split):
    m = mode | ((kind + 1) << 8) | (split << 16)
    rc = rt.lib.cv_gemm_bench(rt.h, M, N, K, ak, bk, m, 20, C.byref(ms))
    return ms.value * 1e3 if rc == 0 else float("nan")
for b in (256, 1024, 2048, 8192):
    shapes = [("jvp0", b, 1024, 785, 1, 0, 1), ("jvp1", b, 1024, 2049, 1, 0, 1), ("dx", b, 1024, 1024, 1, 1, 1),
              ("dw", 1025, 1024, b, 0, 0, 0)]
    for name, M, N, K, ak, bk, mode in shapes:
        auto = t(M, N, K, ak, bk, mode, -1, 0)
        row = [f"{name} b={b} M={M} N={N} K={K}: auto {auto:.1f}"]
        best = (auto, "auto")
        for kind in (1, 2, 3, 5):
            for sp in (1, 2, 4, 8, 16):
                if mode == 1 and sp > 1 and False: pass
                v = t(M, N, K, ak, bk, mode, kind, sp)
                if v == v and v < best[0]: best = (v, f"k{kind}s{sp}")
                row.append(f"k{kind}s{sp} {v:.1f}")
        print(" | ".join(row), "|| best", best, flush=True)
