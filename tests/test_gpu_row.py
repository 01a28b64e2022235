"""GPU parity of the row-space lane beyond the golden primitives:

* the row-space CG lane (egn_mse_cg; method.py:270-282 -> solvers.py:164-174) through
  Method.step against the reference's own trajectory (tests/golden/rowcg.npz), and one
  row_solve_cg on a snapshot Gram;
* the native dense solves on a caller-owned Gram (cv_dense_cholesky_solve /
  cv_dense_cg_solve), incl. partial panels and the not-PD contract error;
* the SYRK-built Gram is exactly symmetric;
* the two-level Cholesky at m = 10,240 (b = 1024, 784-1024-1024-10 CE): the backprojected
  direction against the mask-matched f64 oracle within 1e-4.
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
    b = b.detach().double().cpu().numpy() if hasattr(b, "detach") else np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a.ravel() - b.ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def _reg_batches(bs, n):
    (Xtr, ytr), _ = O.gen_regression(2000, 32, 0.1, 0)
    root = O.ORng(0)
    w = O.init_params((32, 64, 64, 1), "relu", root.split())
    bat = O.Batcher(Xtr, ytr, bs, root.split())
    return w, [bat.next() for _ in range(n)]


def test_row_cg_lane_trajectory_vs_reference(golden):
    g = golden("rowcg")
    w0, batches = _reg_batches(96, 5)
    model = P.Model(32, (64, 64), 1, "relu")
    meth = P.make("egn_mse_cg", model)
    w = P.ParamVector(w0, P.models.param_layout(model))
    st = meth.init(w, seed=0)
    rows = []
    for X, y in batches:
        w, st, info = meth.step(w, P.Batch(X, y, "mse"), st)
        rows.append(info.to_row())
    rows = np.array(rows, dtype=np.float64)
    ref = g["egn_mse_cg/info"]
    assert np.array_equal(np.isnan(rows), np.isnan(ref))
    F = P.STEP_INFO_FIELDS
    for f in ("solver_iterations", "solver_converged", "step_index"):
        assert np.array_equal(rows[:, F.index(f)], ref[:, F.index(f)]), f
    for f in ("loss_before", "grad_norm", "step_norm", "lam"):
        np.testing.assert_allclose(rows[:, F.index(f)], ref[:, F.index(f)], rtol=REL, err_msg=f)
    # the residual after maxiter = 5 iterations of an fp32 recurrence vs f64
    np.testing.assert_allclose(rows[:, F.index("final_relative_residual")], ref[:, F.index("final_relative_residual")],
                               rtol=2e-2)
    assert rel(w.data, g["egn_mse_cg/w_final"]) < REL


def test_row_solve_cg_on_snapshot_gram(golden):
    g = golden("rowcg")
    w0, batches = _reg_batches(96, 1)
    model = P.Model(32, (64, 64), 1, "relu")
    snap = P.make_snapshot("ggn_mse", model, P.ParamVector(w0, P.models.param_layout(model)), P.Batch(*batches[0], "mse"))
    cfg = P.CgConfig(tol=1e-5, maxiter=10, stabilise_every=10, warm_start=True)
    v, it, conv, rr = P.solvers.row_solve_cg(snap.row.gram_matvec, snap.row.rhs, 96.0, cfg)
    assert rel(v, g["solve/v"]) < REL
    assert it == int(g["solve/stats"][0]) and int(conv) == int(g["solve/stats"][1])
    # the dense form (the reference's own `lambda u: gram @ u` over the materialised Gram)
    v2, it2, _, _ = P.solvers.row_solve_cg(snap.row.gram(), snap.row.rhs, 96.0, cfg)
    assert it2 == it and rel(v2, v) < 1e-6
    snap.close()


@pytest.mark.parametrize("m", [200, 1500])
def test_dense_solves_on_a_caller_gram(m):
    rng = np.random.default_rng(m)
    J = rng.standard_normal((m, m // 2 + 7))
    G = J @ J.T / J.shape[1]
    r = rng.standard_normal(m)
    mu = 0.5
    v = P.solvers.row_solve_cholesky(torch.tensor(G, dtype=torch.float32, device="cuda"), r, mu)
    ref = np.linalg.solve(G.astype(np.float32).astype(np.float64) + mu * np.eye(m), r.astype(np.float32))
    assert rel(v, ref) < 1e-6
    cfg = P.CgConfig(tol=1e-6, maxiter=40, stabilise_every=10)
    Gt = torch.tensor(G, dtype=torch.float32, device="cuda")
    x, it, conv, rr = P.solvers.row_solve_cg(Gt, r, mu, cfg)
    o = O.cg(lambda u: G @ u, r, mu, tol=1e-6, maxiter=40, stabilise_every=10)
    assert abs(it - o.iterations) <= 1
    assert rel(x, o.x) < 1e-4
    with pytest.raises(P.ContractError, match="not positive definite"):
        P.solvers.row_solve_cholesky(Gt, r, -10.0)


def test_syrk_gram_is_exactly_symmetric():
    dims, b = (64, 128, 96, 10), 256
    m = P.Model(dims[0], dims[1:-1], dims[-1], "relu")
    w = P.init_params(m, P.Rng(0))
    X, y = O.synthetic_batch(b, dims[0], dims[-1])
    snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
    G = snap.row.gram()
    assert torch.equal(G, G.T)
    snap.close()


def test_row_cholesky_m10240_direction_vs_oracle():
    dims, b = (784, 1024, 1024, 10), 1024
    m = P.Model(dims[0], dims[1:-1], dims[-1], "relu")
    w = P.init_params(m, P.Rng(0))
    X, y = O.synthetic_batch(b, dims[0], dims[-1])
    snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
    mu = float(b)
    v = snap.row.solve_cholesky(mu)
    d = snap.row.scaled_row_transpose(v).data
    masks = [(snap.activation(l) > 0).cpu().numpy() for l in range(1, len(dims) - 1)]
    lin = O.linearize(dims, "relu", "ce", w.data.cpu().numpy().astype(np.float64) if hasattr(w.data, "cpu") else w.data,
                      X, y, masks=masks)
    seeds, orhs = O.row_seeds_rhs(lin)
    ov = O.row_cholesky(O.output_gram(lin, seeds), orhs, mu)
    e_dir = rel(d, O.row_transpose(lin, seeds, ov))
    print(f"m={b * dims[-1]}: direction vs oracle {e_dir:.2e}")
    assert e_dir < REL
    snap.close()


def test_row_cholesky_lookahead_system_residual():
    """m = 25,600 (b = 2560): large enough that the factorization runs the look-ahead
    (the next panel's diagonal block factored on a side stream beside the trailing update)
    and 1024-wide panels with a partial last panel; the solve must match an fp64 solve of
    the same fp32 Gram (cuSOLVER as the checker)."""
    dims, b = (256, 512, 512, 10), 2560
    m = P.Model(dims[0], dims[1:-1], dims[-1], "relu")
    w = P.init_params(m, P.Rng(0))
    X, y = O.synthetic_batch(b, dims[0], dims[-1])
    snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
    mu = float(b)
    v = snap.row.solve_cholesky(mu).double()
    G = snap.row.gram().double()
    G.diagonal().add_(mu)
    ref = torch.linalg.solve(G, snap.row.rhs.double())
    e = float(torch.linalg.vector_norm(v - ref) / torch.linalg.vector_norm(ref))
    print(f"m={b * dims[-1]}: system {e:.2e}")
    assert e < 1e-6
    del G
    snap.close()


def _dist_solve(snap, mu, rhs=None):
    rt = snap.rt
    r = snap.row.rhs if rhs is None else rhs
    out = torch.empty(r.numel(), dtype=torch.float32, device=rt.device)
    rt.bind_stream()
    rt.call("cv_row_solve_cholesky_dist", rt.h, snap.h, float(mu), r.data_ptr(), out.data_ptr())
    return out


@pytest.mark.parametrize("b", [60, 300, 1024, 2560])
def test_distributed_row_cholesky_on_one_rank(b):
    """cv_row_solve_cholesky_dist on a one-rank context (no collectives): Gram strips,
    panel-column buffer, per-panel trailing updates with look-ahead and the replicated-
    vector solves must give the single-GPU solve (m = 600: one partial panel; 3000: a
    partial last panel; 25,600: 25 panels with look-ahead)."""
    dims = (256, 512, 512, 10)
    m = P.Model(dims[0], dims[1:-1], dims[-1], "relu")
    w = P.init_params(m, P.Rng(0))
    X, y = O.synthetic_batch(b, dims[0], dims[-1])
    snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
    mu = float(b)
    v1 = snap.row.solve_cholesky(mu)
    vd = _dist_solve(snap, mu)
    e = rel(vd, v1)
    print(f"m={b * dims[-1]}: distributed vs single-GPU solve {e:.2e}")
    assert e < 1e-6
    with pytest.raises(P.ContractError, match="not positive definite"):
        _dist_solve(snap, -1e6)
    snap.close()


def test_distributed_row_cg_on_one_rank():
    """cv_row_solve_cg_dist on a one-rank context: the Gram products from the strips
    (row part + transposed strictly-lower part) must reproduce the single-GPU row CG."""
    dims, b = (256, 512, 512, 10), 300
    m = P.Model(dims[0], dims[1:-1], dims[-1], "relu")
    w = P.init_params(m, P.Rng(0))
    X, y = O.synthetic_batch(b, dims[0], dims[-1])
    snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
    cfg = P.CgConfig(tol=1e-8, maxiter=25)
    v1, st1 = snap.row.solve_cg(float(b), cfg)
    rt = snap.rt
    out = torch.empty_like(v1)
    st = torch.empty_like(st1)
    rt.call("cv_row_solve_cg_dist", rt.h, snap.h, float(b), snap.row.rhs.data_ptr(), 1e-8, 25, 10, None,
            out.data_ptr(), st.data_ptr())
    e = rel(out, v1)
    print(f"distributed row CG vs single-GPU: {e:.2e}")
    assert e < 1e-6
    snap.close()
