"""GPU checks of paths the reduced golden cases do not reach.

* The row lane's two-level Cholesky with tensor-core trailing updates (512-column panels)
  only engages for m = b*c > 512; here m = 2560 (5 panels).
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2603_25976_b200 as P  # noqa: E402
from oracle import curvopt_oracle as O  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    a = a.detach().double().cpu().numpy() if hasattr(a, "detach") else np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a.ravel() - b.ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def test_row_cholesky_tensor_panels():
    """(Gram + mu I) v = rhs at m = 2560: the device factorization (TC trailing updates,
    fp64 refinement) solves the device's own fp32 system to fp64-level accuracy, and the
    backprojected direction matches the oracle's row lane."""
    dims, b = (64, 128, 96, 10), 256
    m = P.Model(dims[0], dims[1:-1], dims[-1], "relu")
    w = P.init_params(m, P.Rng(0))
    X, y = O.synthetic_batch(b, dims[0], dims[-1])
    snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
    mu = float(b)  # damping_to_row: mu = b * lam, lam = 1
    G = snap.row.gram().double().cpu().numpy()
    r = snap.row.rhs.double().cpu().numpy()
    v = snap.row.solve_cholesky(mu)
    v_ref = np.linalg.solve(G + mu * np.eye(G.shape[0]), r)
    e_sys = rel(v, v_ref)
    masks = [(snap.activation(l) > 0).cpu().numpy() for l in range(1, len(dims) - 1)]
    lin = O.linearize(dims, "relu", "ce", w.data, X, y, masks=masks)
    seeds, orhs = O.row_seeds_rhs(lin)
    ov = O.row_cholesky(O.output_gram(lin, seeds), orhs, mu)
    e_dir = rel(snap.row.scaled_row_transpose(v).data, O.row_transpose(lin, seeds, ov))
    print(f"m={G.shape[0]}: system {e_sys:.2e}, direction vs oracle {e_dir:.2e}")
    assert e_sys < 1e-6
    assert e_dir < 1e-4
    snap.close()
