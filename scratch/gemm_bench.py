import sys, ctypes as C
sys.path.insert(0, ".")
import torch
import paper_2603_25976_b200 as P
from paper_2603_25976_b200.runtime import runtime
rt = runtime()
shapes = [("JVP0", 8192, 1024, 785, 1, 0, 1), ("JVP1 (1seg K=2049)", 8192, 1024, 2049, 1, 0, 1),
          ("dX1", 8192, 1024, 1024, 1, 1, 1), ("dW1", 1025, 1024, 8192, 0, 0, 0),
          ("JVP0 store", 8192, 1024, 785, 1, 0, 0), ("dX1 store", 8192, 1024, 1024, 1, 1, 0),
          ("big 8192^2x1024", 8192, 8192, 1024, 1, 1, 0), ("big split", 8192, 8192, 1024, 1, 1, 1)]
for name, M, N, K, ak, bk, mode in shapes:
    ms = C.c_float()
    rt.call("cv_gemm_bench", rt.h, M, N, K, ak, bk, mode, 20, C.byref(ms))
    fl = 2.0 * M * N * K
    print(f"{name:22s} {M}x{N}x{K} a_km={ak} b_km={bk} mode={mode}: {ms.value*1e3:8.1f} us  "
          f"{fl/ms.value/1e9:7.1f} TF/s useful  {3*fl/ms.value/1e9:7.1f} TF/s fp16")
