"""The tcgen05 3xTF32 engine against the exact-fp32 SIMT engine on the same
snapshot: every GEMM shape of the linearization, GGN product and HVP."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2603_25976_b200 as P  # noqa: E402
from paper_2603_25976_b200.runtime import runtime  # noqa: E402


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm())


# tanh nets compare tightly; relu nets can take a different branch at a kink when
# the two engines differ by ~1e-7 in a pre-activation, hence the looser bound.
SHAPES = [
    ((784, 128, 10), 128, "relu", "ce"),
    ((784, 1024, 1024, 10), 256, "tanh", "ce"),
    ((784, 1024, 1024, 10), 256, "relu", "ce"),
    ((256, 512, 384, 10), 200, "tanh", "mse"),
    ((3072, 512, 512, 10), 96, "tanh", "ce"),
]


@pytest.mark.parametrize("dims,b,act,loss", SHAPES)
def test_tc_matches_simt(dims, b, act, loss):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rt = runtime()
    m = P.Model(dims[0], dims[1:-1], dims[-1], act)
    w = P.init_params(m, P.Rng(0))
    r = P.Rng(1)
    X = r.normal(b * dims[0]).reshape(b, dims[0])
    y = r.integers(b, dims[-1]) if loss == "ce" else r.normal(b * dims[-1]).reshape(b, dims[-1])
    batch = P.Batch(X, y, loss)
    v = P.ParamVector(P.Rng(2).normal(w.dim), w.layout)
    out = {}
    for eng in ("simt", "tc"):
        rt.set_engine(eng if eng == "simt" else "auto")
        snap = P.make_snapshot("ggn_ce" if loss == "ce" else "ggn_mse", m, w, batch)
        out[eng] = (snap.grad.data.clone(), snap.matvec(v).data.clone(), snap.hvp(v).data.clone(),
                    snap.loss_before)
        snap.close()
    rt.set_engine("auto")
    g_s, gv_s, hv_s, l_s = out["simt"]
    g_t, gv_t, hv_t, l_t = out["tc"]
    # The tensor core truncates inside each 8-product tf32 block (measured: -8e-7
    # relative bias per GEMM output); weight gradients sum b
    # per-example terms that largely cancel, which amplifies that ~20-40x.
    tol = 5e-5 if act == "tanh" or len(dims) == 3 else 2e-4
    assert abs(l_s - l_t) <= 1e-5 * abs(l_s)
    assert rel(g_t, g_s) < tol, rel(g_t, g_s)
    assert rel(gv_t, gv_s) < tol, rel(gv_t, gv_s)
    assert rel(hv_t, hv_s) < tol, rel(hv_t, hv_s)


def _gemm(engine, M, N, K, a_km, b_km, seed=0):
    rt = runtime()
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = torch.randn(M, K, device="cuda", generator=g)
    B = torch.randn(K, N, device="cuda", generator=g)
    a = A.contiguous() if a_km else A.t().contiguous()      # K-major: row m holds A[m, :]
    b = B.t().contiguous() if b_km else B.contiguous()      # K-major: row n holds B[:, n]
    lda = K if a_km else M
    ldb = K if b_km else N
    out = torch.full((M, N), float("nan"), device="cuda")
    from paper_2603_25976_b200 import _lib
    rt.call("cv_gemm_test", rt.h, _lib.ENGINE[engine], M, N, K, a.data_ptr(), lda, int(a_km), b.data_ptr(), ldb,
            int(b_km), out.data_ptr(), N)
    ref = A.double() @ B.double()
    return out, ref


@pytest.mark.parametrize("a_km", [1, 0])
@pytest.mark.parametrize("b_km", [1, 0])
@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (256, 512, 96), (200, 300, 70), (200, 296, 72),
                                   (1024, 1024, 1024), (8192, 1024, 785)])
def test_gemm_unit(a_km, b_km, M, N, K):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if (not a_km and M % 8) or (not b_km and N % 8) or (a_km and K % 8) or (b_km and K % 8):
        pytest.skip("leading dimension not 16-byte aligned (fp16 rows)")
    out, ref = _gemm("tc", M, N, K, a_km, b_km)
    err = float((out.double() - ref).norm() / ref.norm())
    assert err < 1e-5, (err, out[:2, :4].tolist(), ref[:2, :4].tolist())


@pytest.mark.parametrize("s2", [1.0, 2.0 ** -7, 2.0 ** 9, 2.0 ** -20, 2.0 ** 23, 2.0 ** -40])
@pytest.mark.parametrize("M,N,K", [(256, 256, 512), (8192, 1024, 256), (200, 48, 72)])
def test_two_segment_rescale(s2, M, N, K):
    """Segments with exponents differing by up to 2^40 share one accumulator:
    the larger-scale segment runs first and is rescaled (scale-input-d, plus
    zero-operand MMAs beyond 2^15) before the second accumulates."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rt = runtime()
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn(M, K, device="cuda", generator=g)
    B = torch.randn(N, K, device="cuda", generator=g)
    out = torch.full((M, N), float("nan"), device="cuda")
    rt.call("cv_gemm_test_seg2", rt.h, M, N, K, A.data_ptr(), B.data_ptr(), float(s2), out.data_ptr())
    ref = (1.0 + s2) * (A.double() @ B.double().t())
    err = float((out.double() - ref).norm() / ref.norm())
    assert err < 2e-6, err
