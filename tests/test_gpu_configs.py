"""Parity at the architectures of BASELINE configs[3] (C4: 3072-2048-2048-10, row lane) and
configs[4] (C5: 3072-4096x4-10, exact-Hessian products) at batches the f64 oracle finishes
in seconds; the full-batch sizes are covered by size-independent properties elsewhere
(C4 lane residual, C5 HVP timing) -- see DESIGN §2 / §6.4."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2603_25976_b200 as P  # noqa: E402
from oracle import curvopt_oracle as O  # noqa: E402

REL = 1e-4


def rel(a, b):
    a = a.detach().double().cpu().numpy() if hasattr(a, "detach") else np.asarray(a, dtype=np.float64)
    b = b.detach().double().cpu().numpy() if hasattr(b, "detach") else np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a.ravel() - b.ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def _matched(dims, snap, w, X, y):
    masks = [(snap.activation(l) > 0).cpu().numpy() for l in range(1, len(dims) - 1)]
    wd = w.data.cpu().numpy() if hasattr(w.data, "cpu") else w.data
    return O.linearize(dims, "relu", "ce", np.asarray(wd, dtype=np.float64), X, y, masks=masks)


def test_c5_architecture_products_vs_oracle():
    """3072-4096x4-10 (d = 63M) at b = 128: exact-Hessian and GGN products, loss and
    gradient against the oracle with the device's ReLU masks; operator symmetry."""
    dims = (3072, 4096, 4096, 4096, 4096, 10)
    m = P.Model(dims[0], dims[1:-1], dims[-1], "relu")
    w = P.init_params(m, P.Rng(0))
    X, y = O.synthetic_batch(128, dims[0], dims[-1])
    snap = P.make_snapshot("hessian", m, w, P.Batch(X, y, "ce"))
    lin = _matched(dims, snap, w, X, y)
    assert snap.loss_before == pytest.approx(lin.value, rel=1e-5)
    assert rel(snap.grad.data, lin.grad) < REL
    v = O.ORng(2).normal(w.dim)
    hv = snap.hvp(P.ParamVector(v, w.layout)).data
    e_h = rel(hv, O.hvp(lin, v))
    e_g = rel(snap.ggn(P.ParamVector(v, w.layout)).data, O.ggn_matvec(lin, v))
    print(f"C5 architecture, b=128: HVP {e_h:.2e}, GGN {e_g:.2e}")
    assert e_h < REL and e_g < REL
    u = O.ORng(3).normal(w.dim)
    hu = snap.hvp(P.ParamVector(u, w.layout)).data.double().cpu().numpy()
    hvn = hv.double().cpu().numpy()
    assert abs(u @ hvn - v @ hu) <= 1e-5 * abs(u @ hvn)
    snap.close()


def test_c4_architecture_row_lane_vs_oracle():
    """3072-2048-2048-10 at b = 256 (m = 2560: two full 1024-row panels and a partial one):
    the row-lane direction (Gram SYRK, panel Cholesky with look-ahead, refinement,
    back-projection) against the oracle's Gram + Cholesky with the device's masks."""
    dims = (3072, 2048, 2048, 10)
    m = P.Model(dims[0], dims[1:-1], dims[-1], "relu")
    w = P.init_params(m, P.Rng(0))
    b = 256
    X, y = O.synthetic_batch(b, dims[0], dims[-1])
    snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
    lin = _matched(dims, snap, w, X, y)
    mu = float(b)
    d = snap.row.scaled_row_transpose(snap.row.solve_cholesky(mu)).data
    seeds, orhs = O.row_seeds_rhs(lin)
    ov = O.row_cholesky(O.output_gram(lin, seeds), orhs, mu)
    e = rel(d, O.row_transpose(lin, seeds, ov))
    print(f"C4 architecture, b=256: row-lane direction vs oracle {e:.2e}")
    assert e < REL
    snap.close()
