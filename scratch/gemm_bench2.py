import sys, os, ctypes as C, subprocess
sys.path.insert(0, ".")
import paper_2603_25976_b200 as P
from paper_2603_25976_b200.runtime import runtime
rt = runtime()
shapes = [("dW0", 785, 1024, 8192, 0, 0, 0), ("dW1", 1025, 1024, 8192, 0, 0, 0), ("JVP0", 8192, 1024, 785, 1, 0, 1),
          ("dX1", 8192, 1024, 1024, 1, 1, 1), ("JVP1-like", 8192, 1024, 2049, 1, 0, 1)]
for name, M, N, K, ak, bk, mode in shapes:
    ms = C.c_float()
    rt.call("cv_gemm_bench", rt.h, M, N, K, ak, bk, mode, 20, C.byref(ms))
    print(f"{os.environ.get('CURVOPT_TC_KIND','auto'):4s} {name:10s} {ms.value*1e3:8.1f} us")
