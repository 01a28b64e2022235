"""Pin the CPU oracle (oracle/curvopt_oracle.py) against fixtures produced by
the real reference (tests/golden/make_golden.py).  CPU only."""

import math

import numpy as np
import pytest

from oracle import curvopt_oracle as O


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def test_rng_streams_bit_exact(golden):
    g = golden("rng")
    for i in range(4):
        s, c, n = (int(x) for x in g[f"case{i}"])
        assert np.array_equal(O.ORng(s, c).raw(n), g[f"raw{i}"])
        assert np.array_equal(O.rademacher(O.ORng(s, c), n), g[f"rad{i}"])
        assert np.array_equal(O.ORng(s, c).uniform(n), g[f"uni{i}"])
        assert np.array_equal(O.ORng(s, c).normal(n + 1), g[f"nrm{i}"])
        assert np.array_equal(O.ORng(s, c).integers(n, 10), g[f"int{i}"])
        assert np.array_equal(O.ORng(s, c).permutation(min(n, 500)), g[f"perm{i}"])
        assert O.ORng(s, c).split().seed == int(g[f"split{i}"][0])


NAMES = ["relu_ce", "tanh_ce", "relu_mse", "tanh_mse", "lin_ce"]


@pytest.mark.parametrize("name", NAMES)
def test_primitives_match_reference(golden, name):
    g = golden("primitives")
    k = lambda s: g[f"{name}/{s}"]  # noqa: E731
    dims = tuple(int(x) for x in k("dims"))
    act, loss = str(k("act")), str(k("loss"))
    w = k("w")
    assert np.array_equal(w, O.init_params(dims, act, O.ORng(0)))
    lin = O.linearize(dims, act, loss, w, k("X"), k("y"))
    assert lin.value == pytest.approx(float(k("value")), rel=1e-13)
    assert rel(lin.grad, k("grad")) < 1e-12
    assert rel(lin.out, k("out")) < 1e-12
    v = k("v")
    assert rel(O.jvp(lin, v), k("jvp")) < 1e-12
    assert rel(O.vjp(lin, k("U")), k("vjp")) < 1e-12
    assert rel(O.ggn_matvec(lin, v), k("ggn")) < 1e-12
    assert rel(O.hvp(lin, v), k("hvp")) < 1e-12
    mv = lambda x: O.ggn_matvec(lin, x)  # noqa: E731
    res = O.cg(mv, lin.grad, 0.5, 1e-5, 10, 3)
    st = k("cg_stats")
    assert rel(res.x, k("cg_x")) < 1e-10
    assert (res.iterations, int(res.converged), int(res.negative_curvature)) == (int(st[0]), int(st[1]), int(st[3]))
    assert res.relres == pytest.approx(st[2], rel=1e-8)
    res = O.cg(mv, lin.grad, 0.5, 1e-5, 10, 3, precond=k("pcg_pre"), x0=k("pcg_x0"))
    st = k("pcg_stats")
    assert rel(res.x, k("pcg_x")) < 1e-10
    assert (res.iterations, int(res.converged)) == (int(st[0]), int(st[1]))
    rng = O.ORng(5)
    d = w.size
    assert rel(O.hutchinson_diag(mv, rng, d, 3), k("hutch_diag")) < 1e-12
    assert O.hutchinson_trace(mv, rng, d, 2) == pytest.approx(float(k("hutch_trace")), rel=1e-12)
    assert O.power_iter_top_eig(mv, rng, d, 7) == pytest.approx(float(k("top_eig")), rel=1e-10)
    assert rng.counter == int(k("rng_after")[0])
    seeds, rhs = O.row_seeds_rhs(lin)
    assert rel(seeds, k("seeds")) < 1e-10
    assert rel(rhs, k("rhs")) < 1e-10
    gram = O.output_gram(lin, seeds)
    assert rel(gram, k("gram")) < 1e-10
    vrow = O.row_cholesky(gram, rhs, float(k("mu")))
    assert rel(O.row_transpose(lin, seeds, vrow), k("rowdir")) < 1e-9
    la = O.loss_value(dims, act, loss, w + 0.01 * v, k("X"), k("y"))
    assert la == pytest.approx(float(k("loss_at")), rel=1e-13)


def _cmp_rows(mine, ref, tol=1e-9):
    mine = np.asarray(mine, dtype=np.float64)
    assert mine.shape == ref.shape
    nan_m, nan_r = np.isnan(mine), np.isnan(ref)
    assert np.array_equal(nan_m, nan_r), "sentinel placement differs"
    ok = ~nan_r
    np.testing.assert_allclose(mine[ok], ref[ok], rtol=tol, atol=1e-12)


def _run(spec, dims, act, loss, w, batches, seed=0):
    st = O.oracle_init(spec, w.size, seed)
    rows = []
    for X, y in batches:
        w, st, info, _ = O.oracle_step(spec, dims, act, loss, w, X, y, st)
        rows.append([info[f] for f in O.STEP_FIELDS])
    return np.array(rows, dtype=np.float64), w


def test_c1_planned_step(golden):
    g = golden("trajectories")
    dims = (784, 128, 10)
    w = O.init_params(dims, "relu", O.ORng(0))
    X, y = O.synthetic_batch(128, 784, 10)
    spec = O.OSpec()
    st = O.oracle_init(spec, w.size)
    w1, st, info, direction = O.oracle_step(spec, dims, "relu", "ce", w, X, y, st)
    _cmp_rows([info[f] for f in O.STEP_FIELDS], g["c1/info0"])
    assert rel(direction, g["c1/direction"]) < 1e-6
    w2, st, info, _ = O.oracle_step(spec, dims, "relu", "ce", w1, X, y, st)
    _cmp_rows([info[f] for f in O.STEP_FIELDS], g["c1/info1"])


def test_c2_trajectory_100_steps(golden):
    g = golden("trajectories")
    dims = (784, 128, 10)
    (Xtr, ytr), _ = O.gen_classification(20000, 784, 10, 10.0, 0)
    bat = O.Batcher(Xtr, ytr, 128, O.ORng(0).split())
    batches = [bat.next() for _ in range(100)]
    assert float(batches[0][0].sum()) == pytest.approx(float(g["c2/first_batch_idx_sum"]), rel=1e-14)
    spec = O.OSpec(damping="trust_region", tr_every_k=5, estimator_every_k=10)
    w = O.init_params(dims, "relu", O.ORng(0))
    rows, wf = _run(spec, dims, "relu", "ce", w, batches)
    _cmp_rows(rows, g["c2/info"], tol=1e-8)
    assert np.linalg.norm(wf) == pytest.approx(float(g["c2/w_final_norm"]), rel=1e-10)


def test_c3_reduced_pcg(golden):
    g = golden("trajectories")
    dims = (784, 1024, 1024, 10)
    w = O.init_params(dims, "relu", O.ORng(0))
    X, y = O.synthetic_batch(256, 784, 10)
    spec = O.OSpec(precond="diag_ema", estimator_every_k=2)
    rows, wf = _run(spec, dims, "relu", "ce", w, [(X, y)] * 3)
    _cmp_rows(rows, g["c3r/info"], tol=1e-8)


def test_c4_reduced_row_lane(golden):
    g = golden("trajectories")
    dims = (96, 64, 64, 10)
    w = O.init_params(dims, "relu", O.ORng(0))
    X, y = O.synthetic_batch(32, 96, 10)
    rows, wf = _run(O.OSpec(solver="row_cholesky"), dims, "relu", "ce", w, [(X, y)] * 2)
    _cmp_rows(rows, g["c4r/info"], tol=1e-8)
    assert rel(wf, g["c4r/w_final"]) < 1e-12


def test_c5_reduced_hessian(golden):
    g = golden("trajectories")
    dims = (48, 32, 32, 32, 32, 10)
    w = O.init_params(dims, "relu", O.ORng(0))
    X, y = O.synthetic_batch(64, 48, 10)
    spec = O.OSpec(curvature="hessian", estimator_every_k=1, trace_every_k=1, trace_probes=2, rho_every_k=2)
    rows, wf = _run(spec, dims, "relu", "ce", w, [(X, y)] * 3)
    _cmp_rows(rows, g["c5r/info"], tol=1e-8)
    assert rel(wf, g["c5r/w_final"]) < 1e-12


TC_NAMES = ["relu_ce", "tanh_ce", "relu_mse", "tanh_mse"]


@pytest.mark.parametrize("name", TC_NAMES)
def test_tensor_core_sized_primitives_match_reference(golden, name):
    """The b >= 128 fixtures the GPU parity tests run on the tensor-core engine."""
    g = golden("primitives_tc")
    k = lambda s: g[f"{name}/{s}"]  # noqa: E731
    dims = tuple(int(x) for x in k("dims"))
    act, loss = str(k("act")), str(k("loss"))
    w = k("w")
    assert np.array_equal(w, O.init_params(dims, act, O.ORng(0)))
    X, y = O.synthetic_batch(k("X").shape[0], dims[0], dims[-1], loss=loss)
    assert np.array_equal(X, k("X"))
    lin = O.linearize(dims, act, loss, w, X, y)
    assert lin.value == pytest.approx(float(k("value")), rel=1e-13)
    assert rel(lin.grad, k("grad")) < 1e-12
    v = k("v")
    assert rel(O.jvp(lin, v), k("jvp")) < 1e-12
    assert rel(O.vjp(lin, k("U")), k("vjp")) < 1e-12
    assert rel(O.ggn_matvec(lin, v), k("ggn")) < 1e-12
    assert rel(O.hvp(lin, v), k("hvp")) < 1e-12
    res = O.cg(lambda x: O.ggn_matvec(lin, x), lin.grad, 0.5, 1e-5, 10, 3)
    assert rel(res.x, k("cg_x")) < 1e-10 and res.iterations == int(k("cg_stats")[0])
    res = O.cg(lambda x: O.hvp(lin, x), lin.grad, 2.0, 1e-5, 10, 3)
    st = k("hcg_stats")
    assert rel(res.x, k("hcg_x")) < 1e-9
    assert (res.iterations, int(res.converged), int(res.negative_curvature)) == (int(st[0]), int(st[1]), int(st[3]))
    rng = O.ORng(5)
    mv = lambda x: O.ggn_matvec(lin, x)  # noqa: E731
    assert rel(O.hutchinson_diag(mv, rng, w.size, 2), k("hutch_diag")) < 1e-12
    assert O.hutchinson_trace(mv, rng, w.size, 2) == pytest.approx(float(k("hutch_trace")), rel=1e-12)


CHAINS = {
    "sophia": (("trace_momentum", {"beta": 0.96}), ("sophia_clip", {"gamma": 0.05, "eps": 1e-12}),
               ("add_decayed_weights", {"weight_decay": 1e-4}),
               ("scale_by_schedule", {"schedule": "constant", "alpha0": 0.01}), ("scale", {"value": -1.0})),
    "adam": (("scale_by_adam", {"b1": 0.9, "b2": 0.999, "eps": 1e-8}),
             ("scale_by_schedule", {"schedule": "constant", "alpha0": 1e-3}), ("scale", {"value": -1.0})),
    "sgdm": (("trace_momentum", {"beta": 0.9}), ("add_decayed_weights", {"weight_decay": 5e-4}),
             ("scale_by_schedule", {"schedule": "constant", "alpha0": 0.05}), ("scale", {"value": -1.0})),
    "clip_cos": (("clip_global_norm", {"max_norm": 0.5}),
                 ("scale_by_schedule", {"schedule": "cosine_warmup", "alpha0": 0.3, "warmup": 2, "total": 6}),
                 ("trace_momentum", {"beta": 0.5}), ("clip_global_norm", {"max_norm": 0.05}),
                 ("scale", {"value": -2.0})),
    "step_decay": (("scale_by_schedule", {"schedule": "step_decay", "alpha0": 0.2, "gamma": 0.5, "period": 2}),
                   ("scale", {"value": -1.0})),
}


@pytest.mark.parametrize("name", list(CHAINS))
def test_chain_links_match_reference(golden, name):
    g = golden("chains")
    d = 3001
    w = O.ORng(11).normal(d)
    assert np.array_equal(w, g[f"{name}/w0"])
    pre = np.abs(O.ORng(12).normal(d)) * 1e-2
    chain = CHAINS[name]
    st = O.chain_init(chain, d)
    for t in range(4):
        direc = O.ORng(20 + t).normal(d) * (3.0 if t == 1 else 1.0)
        upd, st = O.chain_apply(chain, st, direc, w, t, pre)
        assert rel(upd, g[f"{name}/upd{t}"]) < 1e-13
        for i, s in enumerate(st):
            for key, val in s.items():
                assert rel(np.asarray(val, dtype=np.float64), g[f"{name}/st{t}_{i}_{key}"]) < 1e-13
        w = w + upd


def test_gnb_diag_matches_reference(golden):
    g = golden("gnb_presets")
    dims = (64, 96, 64, 10)
    w = O.init_params(dims, "relu", O.ORng(0))
    X, y = O.synthetic_batch(128, 64, 10)
    lin = O.linearize(dims, "relu", "ce", w, X, y)
    rng = O.ORng(7)
    assert rel(O.gnb_diag(lin, rng, 3), g["gnb/diag"]) < 1e-12
    assert rng.counter == int(g["gnb/rng_after"][0])


@pytest.mark.parametrize("preset", ["sophia_g", "sophia_h", "sophia_n", "adahessian", "adam", "sgdm", "sgd"])
def test_preset_trajectories_match_reference(golden, preset):
    g = golden("gnb_presets")
    dims = (64, 96, 64, 10)
    w = O.init_params(dims, "relu", O.ORng(0))
    spec = O.preset_ospec(preset)
    rows, wf = _run(spec, dims, "relu", "ce", w, [O.synthetic_batch(128, 64, 10, seed=1 + t) for t in range(4)])
    _cmp_rows(rows, g[f"{preset}/info"], tol=1e-9)
    assert rel(wf, g[f"{preset}/w_final"]) < 1e-11


def test_regression_data_and_newton_cg_cadence_run(golden):
    """The cadence study's workload (harness/data.py:49-60, bench.py:135-207)."""
    g = golden("harness")
    (Xtr, ytr), (Xte, yte) = O.gen_regression(2000, 32, 0.1, 0)
    assert float(Xtr.sum()) == pytest.approx(float(g["reg/train_X_sum"]), rel=1e-13)
    assert np.array_equal(ytr[:50, 0], g["reg/train_y"])
    assert Xte.shape[0] == int(g["reg/test_n"])
    root = O.ORng(0)
    dims = (32, 64, 64, 1)
    w = O.init_params(dims, "relu", root.split())
    bat = O.Batcher(Xtr, ytr, 128, root.split())
    batches = [bat.next() for _ in range(6)]
    assert np.array_equal(batches[0][0][:4], g["reg/batch0_idx_X"])
    spec = O.OSpec(curvature="hessian", maxiter=3, rho_every_k=2, chain=(("scale", {"value": 1e-3}),
                                                                        ("scale", {"value": -1.0})))
    rows, wf = _run(spec, dims, "relu", "mse", w, batches)
    _cmp_rows(rows, g["newton_cg/info"], tol=1e-8)
    assert rel(wf, g["newton_cg/w_final"]) < 1e-11


def test_row_cg_lane_matches_reference(golden):
    """egn_mse_cg (method.py:270-282 -> solvers.py:164-174): row-space CG on the Gram,
    warm-started from the previous step's row-space solution."""
    g = golden("rowcg")
    (Xtr, ytr), _ = O.gen_regression(2000, 32, 0.1, 0)
    root = O.ORng(0)
    dims = (32, 64, 64, 1)
    w = O.init_params(dims, "relu", root.split())
    bat = O.Batcher(Xtr, ytr, 96, root.split())
    batches = [bat.next() for _ in range(5)]
    lin = O.linearize(dims, "relu", "mse", w, *batches[0])
    seeds, rhs = O.row_seeds_rhs(lin)
    gram = O.output_gram(lin, seeds)
    res = O.cg(lambda u: gram @ u, rhs, 96.0)
    assert rel(res.x, g["solve/v"]) < 1e-12
    assert [res.iterations, int(res.converged)] == [int(x) for x in g["solve/stats"][:2]]
    spec = O.OSpec(curvature="ggn_mse", solver="row_cg", maxiter=5)
    rows, wf = _run(spec, dims, "relu", "mse", w, batches)
    _cmp_rows(rows, g["egn_mse_cg/info"], tol=1e-8)
    assert rel(wf, g["egn_mse_cg/w_final"]) < 1e-11
