"""The timing harness (paper_2603_25976_b200.harness) against the reference's harness
(curvopt/harness: data.py, run.py, bench.py): datasets and batches bit-exact with the
reference's goldens, the timing summary rule, and on the GPU the cadence study's
workload (newton_cg, constant damping, rho cadence) against the reference run."""

import math

import numpy as np
import pytest

from paper_2603_25976_b200 import harness as H


def test_regression_dataset_matches_reference(golden):
    g = golden("harness")
    tr, te = H.gen_regression(2000, 32, 0.1, 0)
    assert float(tr.X.sum()) == pytest.approx(float(g["reg/train_X_sum"]), rel=1e-13)
    assert np.array_equal(tr.y[:50, 0], g["reg/train_y"])
    assert te.n == int(g["reg/test_n"])
    assert tr.loss_kind == "mse" and tr.y.shape == (1800, 1)


def test_classification_dataset_matches_oracle():
    from oracle import curvopt_oracle as O

    tr, te = H.gen_classification(500, 12, 10, 10.0, 3)
    (oX, oy), (tX, ty) = O.gen_classification(500, 12, 10, 10.0, 3)
    assert np.array_equal(tr.X, oX) and np.array_equal(tr.y, oy) and np.array_equal(te.X, tX)


def test_timing_summary_windows():
    t = [100.0, 100.0] + [1.0] * 50 + [3.0] * 50 + [2.0] * 10
    s = H.timing_summary(t, 2, 50)
    assert s.window_means_ms == (1.0, 3.0, 2.0)
    assert s.median_ms == 2.0 and s.p90_ms == pytest.approx(np.percentile([1.0, 3.0, 2.0], 90))
    assert math.isnan(H.timing_summary([1.0], 2, 5).median_ms)
    with pytest.raises(H.ContractError):
        H.TimingConfig(warmup_steps=0)


def test_cadence_methods_plan():
    import paper_2603_25976_b200 as P

    m = P.Model(16, (32, 32), 1, "relu")
    ms = H.cadence_methods([-1, 2], m)
    assert ms[-1].plan.needs_rho is False and ms[2].plan.needs_rho is True
    assert ms[2].spec.damping.policy == "constant" and ms[2].plan.solver_config.maxiter == 3


@pytest.mark.gpu
def test_newton_cg_cadence_run_vs_reference(golden):
    """harness.npz: newton_cg (hessian + CG maxiter 3, warm start, constant damping,
    rho every 2) on the regression workload, 6 steps, reference vs device."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_25976_b200 as P

    g = golden("harness")
    tr, _ = H.gen_regression(2000, 32, 0.1, 0)
    root = P.Rng(0)
    m = P.Model(32, (64, 64), 1, "relu")
    w = P.init_params(m, root.split()).to_device()
    bat = H.EpochBatcher(tr, 128, root.split())
    meth = P.make("newton_cg", m, damping={"policy": "constant", "lam0": 1.0, "tr": None},
                  solver={"cg": {"maxiter": 3, "warm_start": True}}, telemetry={"rho_every_k": 2})
    st = meth.init(w, seed=0)
    rows = []
    for t in range(6):
        b = bat.next()
        if t == 0:
            assert np.allclose(b.inputs[:4].cpu().numpy(), g["reg/batch0_idx_X"], rtol=1e-6)
        w, st, info = meth.step(w, b, st)
        rows.append(info.to_row())
    rows = np.array(rows, dtype=np.float64)
    ref = g["newton_cg/info"]
    assert np.array_equal(np.isnan(rows), np.isnan(ref))
    F = P.STEP_INFO_FIELDS
    for f in ("solver_iterations", "solver_converged", "step_index"):
        assert np.array_equal(rows[:, F.index(f)], ref[:, F.index(f)]), f
    for f in ("loss_before", "loss_after", "grad_norm", "step_norm"):
        ok = ~np.isnan(ref[:, F.index(f)])
        np.testing.assert_allclose(rows[ok, F.index(f)], ref[ok, F.index(f)], rtol=1e-4, err_msg=f)
    w_ref = g["newton_cg/w_final"]
    assert np.linalg.norm(w.data.double().cpu().numpy() - w_ref) / np.linalg.norm(w_ref) < 1e-4


@pytest.mark.gpu
def test_bench_cadence_paired_protocol():
    """A short cadence study at the paper's shapes: every setting sees the same
    trajectory (identical loss_before per step), rho fields only where the cadence fires."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_25976_b200 as P

    ks = [-1, 10, 5, 2, 1]
    rows, infos = H.bench_cadence(ks, steps=12, window=5, return_infos=True)
    assert [r[0] for r in rows] == ks and all(r[1] > 0 for r in rows)
    F = P.STEP_INFO_FIELDS
    lb = {k: np.array(infos[k])[:, F.index("loss_before")] for k in ks}
    for k in ks[1:]:
        assert np.array_equal(lb[k], lb[-1])
    for k in ks:
        rho = np.array(infos[k])[:, F.index("rho")]
        t = np.arange(len(rho))
        fires = (t % k == 0) if k >= 1 else np.zeros(len(rho), bool)
        assert np.array_equal(~np.isnan(rho), fires)
