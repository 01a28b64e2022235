import sys, ctypes as C
sys.path.insert(0, ".")
import paper_2603_25976_b200 as P
from paper_2603_25976_b200.runtime import runtime
rt = runtime()
M, N, K, ak, bk, mode = (int(x) for x in sys.argv[1:7])
ms = C.c_float()
rt.call("cv_gemm_bench", rt.h, M, N, K, ak, bk, mode, 2, C.byref(ms))
print(ms.value)
