import sys; sys.path.insert(0, ".")
import torch
sys.path.insert(0, "tests")
from test_gemm_engine import _gemm
for K in (64, 256, 1024, 4096, 16384):
    for eng in ("tc", "simt"):
        out, ref = _gemm(eng, 256, 256, K, 1, 1)
        err = float((out.double() - ref).norm() / ref.norm())
        # bias: mean signed relative error
        bias = float(((out.double() - ref) * ref.sign()).mean() / ref.abs().mean())
        print(f"K={K:6d} {eng:5s} rel {err:.2e} bias {bias:+.2e}")
# positive data (no cancellation): error relative to sum
import paper_2603_25976_b200 as P
