"""GPU parity of the fused kernels against the CPU oracle on identical inputs.

The output-layer JVP runs inside the epilogue of the last hidden tangent GEMM
(Epilogue::head_*) whenever that GEMM is on the tensor-core engine: 1-CTA tiles
(hidden width < 256), 2-CTA tiles with a ragged last column tile, the
compile-time c = 10 path and the generic-width path.  Each case checks the GGN
product, the exact HVP and the JVP (the three callers of the fused head) against
the oracle run with the device's ReLU masks (hard part 2).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2603_25976_b200 as P  # noqa: E402
from oracle import curvopt_oracle as O  # noqa: E402

REL = 1e-4


def rel(a, b):
    a = a.detach().double().cpu().numpy() if hasattr(a, "detach") else np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a.ravel() - b.ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


CASES = [
    ((64, 160, 10), 512),           # single hidden layer, 1-CTA 128-wide tiles
    ((96, 256, 160, 10), 512),      # two hidden layers, 1-CTA
    ((100, 512, 384, 10), 1024),    # 2-CTA 256x256 tiles, ragged last column tile
    ((64, 256, 320, 7), 768),       # generic head width (c = 7)
    ((48, 288, 16), 640),           # c = 16 (the widest fused head)
]


@pytest.mark.parametrize("dims,b", CASES)
def test_fused_head_products_vs_oracle(dims, b):
    m = P.Model(dims[0], dims[1:-1], dims[-1], "relu")
    w = P.init_params(m, P.Rng(0))
    X, y = O.synthetic_batch(b, dims[0], dims[-1])
    snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
    masks = [(snap.activation(l) > 0).cpu().numpy() for l in range(1, len(dims) - 1)]
    lin = O.linearize(dims, "relu", "ce", w.data, X, y, masks=masks)
    v = O.ORng(2).normal(w.dim)
    pv = P.ParamVector(v, w.layout)
    e_ggn = rel(snap.matvec(pv).data, O.ggn_matvec(lin, v))
    e_hvp = rel(snap.hvp(pv).data, O.hvp(lin, v))
    e_jvp = rel(snap.jvp(pv), O.jvp(lin, v))
    print(f"{dims} b={b}: ggn {e_ggn:.2e} hvp {e_hvp:.2e} jvp {e_jvp:.2e}")
    assert e_ggn < REL and e_hvp < REL and e_jvp < REL
    snap.close()


def test_fused_head_deterministic():
    """Fixed-order group reduction: two products of the same vector are bit-identical."""
    dims, b = (100, 512, 384, 10), 1024
    m = P.Model(dims[0], dims[1:-1], dims[-1], "relu")
    w = P.init_params(m, P.Rng(0))
    X, y = O.synthetic_batch(b, dims[0], dims[-1])
    snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
    pv = P.ParamVector(O.ORng(5).normal(w.dim), w.layout)
    a = snap.matvec(pv).data.clone()
    c = snap.matvec(pv).data.clone()
    assert torch.equal(a, c)
    snap.close()
