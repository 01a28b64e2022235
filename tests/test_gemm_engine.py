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


SHAPES = [
    ((784, 128, 10), 128, "relu", "ce"),
    ((784, 1024, 1024, 10), 256, "relu", "ce"),
    ((256, 512, 384, 10), 200, "tanh", "mse"),
    ((3072, 512, 512, 10), 96, "relu", "ce"),
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
    assert abs(l_s - l_t) <= 1e-5 * abs(l_s)
    assert rel(g_t, g_s) < 2e-5, rel(g_t, g_s)
    assert rel(gv_t, gv_s) < 2e-5, rel(gv_t, gv_s)
    assert rel(hv_t, hv_s) < 2e-5, rel(hv_t, hv_s)
