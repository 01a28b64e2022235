"""CUDA-graph replay of planned steps (method.StepGraph) is bitwise the eager step:
trajectories with gates that fire on some steps (eager) and not on others (replayed),
trust-region damping (the graph key changes with lam), warm starts and PCG."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2603_25976_b200 as P  # noqa: E402
from oracle import curvopt_oracle as O  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def _run(spec, model, batches, graphs, steps):
    meth = P.assemble(spec, model)
    meth.graphs = graphs
    w = P.init_params(model, P.Rng(0)).to_device()
    st = meth.init(w, 0)
    rows = []
    for t in range(steps):
        X, y = batches[t % len(batches)]
        w, st, info = meth.step(w, P.Batch(X, y, "ce"), st)
        rows.append(info.to_row())
    n_graphs = len(meth._graph_cache)
    meth.release_graphs()
    return np.array(rows, dtype=np.float64), w.data.cpu().numpy(), n_graphs


def _same(a, b):
    return np.array_equal(np.isnan(a), np.isnan(b)) and np.array_equal(a[~np.isnan(a)], b[~np.isnan(b)])


@pytest.mark.parametrize("which", ["pcg_est", "tr_rho"])
def test_graph_replay_bitwise_equals_eager(which):
    model = P.Model(784, (256, 128), 10, "relu")
    batches = [tuple(torch.from_numpy(np.asarray(a)).cuda() for a in O.synthetic_batch(512, 784, 10, seed=1 + i))
               for i in range(3)]
    cg = P.CgConfig(tol=1e-5, maxiter=6, stabilise_every=4, warm_start=True)
    if which == "pcg_est":
        spec = P.MethodSpec(curvature=P.CurvatureSpec("ggn_ce"), solver=P.SolverSpec("cg", cg),
                            precond=P.PrecondSpec("diag_ema", 0.99), damping=P.DampingSpec("constant", 1.0),
                            estimator=P.EstimatorSpec("hutchinson", 1, every_k=3),
                            chain=(P.transforms.scale(1e-3), P.transforms.scale(-1.0)))
    else:
        spec = P.MethodSpec(curvature=P.CurvatureSpec("hessian"), solver=P.SolverSpec("cg", cg),
                            damping=P.DampingSpec("trust_region", 1.0, tr=P.control.TrustRegionConfig(every_k=2)),
                            telemetry=P.TelemetrySpec(rho_every_k=3),
                            chain=(P.transforms.scale(1e-3), P.transforms.scale(-1.0)))
    re, we, _ = _run(spec, model, batches, False, 10)
    rg, wg, ng = _run(spec, model, batches, True, 10)
    assert ng >= 1, "no step was replayed from a graph"
    assert _same(re, rg)
    assert np.array_equal(we, wg)


def test_graph_cache_is_bounded_and_evictions_stay_exact():
    """Six batch shapes in rotation (six graph keys) against a cache of four graphs: the
    least recently used graphs are released and recaptured, and the trajectory is still
    bitwise the eager one."""
    model = P.Model(784, (256, 128), 10, "relu")
    sizes = (128, 192, 256, 320, 384, 448)
    batches = [tuple(torch.from_numpy(np.asarray(a)).cuda() for a in O.synthetic_batch(n, 784, 10, seed=1 + i))
               for i, n in enumerate(sizes)]
    cg = P.CgConfig(tol=1e-5, maxiter=4, warm_start=False)
    spec = P.MethodSpec(curvature=P.CurvatureSpec("ggn_ce"), solver=P.SolverSpec("cg", cg),
                        damping=P.DampingSpec("constant", 1.0), chain=(P.transforms.scale(-1e-3),))

    def run(graphs):
        meth = P.assemble(spec, model)
        meth.graphs = graphs
        w = P.init_params(model, P.Rng(0)).to_device()
        st = meth.init(w, 0)
        rows, live = [], 0
        for t in range(3 * len(sizes) * 2):
            X, y = batches[(t // 2) % len(sizes)]  # each shape twice in a row: seen, then captured
            w, st, info = meth.step(w, P.Batch(X, y, "ce"), st)
            rows.append(info.to_row())
            live = max(live, sum(1 for g in meth._graph_cache.values() if g))
        meth.release_graphs()
        return np.array(rows, dtype=np.float64), w.data.cpu().numpy(), live

    re, we, _ = run(False)
    rg, wg, live = run(True)
    assert 1 <= live <= P.method.Method._MAX_GRAPHS
    assert _same(re, rg)
    assert np.array_equal(we, wg)
