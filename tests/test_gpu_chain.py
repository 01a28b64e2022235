"""Device transform chains (cv_chain_apply), the GNB estimator (cv_gnb_diag) and the
presets built on them, against fixtures produced by the real reference
(tests/golden/make_golden.py: chain_cases, gnb_cases).

Tolerances: fp32 device vectors against f64 reference values; the north star's
1e-4 relative L2 per step for every update, state and estimator output."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2603_25976_b200 as P  # noqa: E402
from oracle import curvopt_oracle as O  # noqa: E402
from paper_2603_25976_b200 import transforms as T  # noqa: E402

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


CHAINS = {
    "sophia": lambda: (T.trace_momentum(0.96), T.sophia_clip(0.05, 1e-12), T.add_decayed_weights(1e-4),
                       T.scale_by_schedule("constant", alpha0=0.01), T.scale(-1.0)),
    "adam": lambda: (T.scale_by_adam(0.9, 0.999, 1e-8), T.scale_by_schedule("constant", alpha0=1e-3), T.scale(-1.0)),
    "sgdm": lambda: (T.trace_momentum(0.9), T.add_decayed_weights(5e-4), T.scale_by_schedule("constant", alpha0=0.05),
                     T.scale(-1.0)),
    "clip_cos": lambda: (T.clip_global_norm(0.5), T.scale_by_schedule("cosine_warmup", alpha0=0.3, warmup=2, total=6),
                         T.trace_momentum(0.5), T.clip_global_norm(0.05), T.scale(-2.0)),
    "step_decay": lambda: (T.scale_by_schedule("step_decay", alpha0=0.2, gamma=0.5, period=2), T.scale(-1.0)),
}


@pytest.mark.parametrize("name", list(CHAINS))
def test_device_chain_matches_reference(golden, name):
    g = golden("chains")
    d = 3001
    lay = (("w", (d,)),)
    dev = torch.device("cuda")
    w = P.ParamVector(torch.tensor(g[f"{name}/w0"], dtype=torch.float32, device=dev), lay)
    pre = P.ParamVector(torch.tensor(g[f"{name}/pre"], dtype=torch.float32, device=dev), lay)
    chain = CHAINS[name]()
    st = P.chain_init(chain, w)
    for t in range(4):
        direc = O.ORng(20 + t).normal(d) * (3.0 if t == 1 else 1.0)
        dv = P.ParamVector(torch.tensor(direc, dtype=torch.float32, device=dev), lay)
        upd, st = P.chain_apply(chain, st, dv, w, t, precond_diag=pre)
        assert upd.data.is_cuda
        assert rel(upd.data, g[f"{name}/upd{t}"]) < REL, (t, rel(upd.data, g[f"{name}/upd{t}"]))
        for i, s in enumerate(st):
            for key, val in s.items():
                ref = g[f"{name}/st{t}_{i}_{key}"]
                if key == "t":
                    assert int(val) == int(ref)
                else:
                    assert rel(val, ref) < REL
        w = P.ParamVector(w.data + upd.data, lay)


def test_chain_step_tail_norms_and_nonfinite():
    """cv_chain_apply's scalars: ||update||, #non-finite (direction, update, w_next), ||direction||^2."""
    from paper_2603_25976_b200.runtime import runtime

    rt = runtime()
    d = 10007
    x = torch.randn(d, device="cuda")
    w = torch.randn(d, device="cuda")
    chain = (T.trace_momentum(0.5), T.clip_global_norm(1.0), T.scale(-3.0))
    st = T.chain_init(chain, P.ParamVector(w, (("w", (d,)),)))
    upd, wn = torch.empty_like(x), torch.empty_like(x)
    scal = torch.zeros(3, dtype=torch.float64, device="cuda")
    T.device_chain_apply(chain, st, x, w, 0, None, rt, upd, wn, scal)
    s = scal.cpu().numpy()
    assert s[0] == pytest.approx(3.0, rel=1e-6)  # clipped to norm 1, then x3
    assert s[1] == 0.0
    assert s[2] == pytest.approx(float((x.double() ** 2).sum()), rel=1e-12)
    assert torch.equal(wn, w + upd)
    x[7] = float("nan")
    T.device_chain_apply(chain, st, x, w, 0, None, rt, upd, wn, scal)
    assert scal[1].item() >= 1.0


def test_gnb_diag_matches_reference(golden):
    g = golden("gnb_presets")
    m = P.Model(64, (96, 64), 10, "relu")
    w = P.init_params(m, P.Rng(0))
    X, y = O.synthetic_batch(128, 64, 10)
    batch = P.Batch(X, y, "ce")
    snap = P.make_snapshot("ggn_ce", m, w, batch)
    rng = P.Rng(7)
    est = P.gnb_diag(m, w, batch, rng, 3, lin=snap)
    assert est.data.is_cuda
    assert rel(est.data, g["gnb/diag"]) < REL, rel(est.data, g["gnb/diag"])
    assert rng.counter == int(g["gnb/rng_after"][0])


def test_gnb_diag_shard_uses_global_uniforms():
    """A shard's label draws are its rows' slice of Rng.uniform(global_size): the two
    half-batch shards draw exactly the labels the full batch draws, so (world = 1, no
    all-reduce) each shard's cotangent rows equal the full batch's rows."""
    m = P.Model(64, (96, 64), 10, "relu")
    w = P.init_params(m, P.Rng(0))
    X, y = O.synthetic_batch(256, 64, 10)
    dims = m.dims
    lin = O.linearize(dims, "relu", "ce", w.data, X, y)
    full = O.gnb_diag(lin, O.ORng(3), 1)
    # the same estimate from the two shards' label draws, assembled on the host
    rng = O.ORng(3)
    u = rng.uniform(256)
    cum = np.cumsum(lin.probs, axis=1)
    labels = np.minimum((u[:, None] > cum).sum(axis=1), 9)
    for half in (0, 1):
        rows = slice(128 * half, 128 * (half + 1))
        b = P.Batch(X[rows], y[rows], "ce", global_size=256, row_offset=128 * half)
        snap = P.make_snapshot("ggn_ce", m, w, b)
        r = P.Rng(3)
        est = P.gnb_diag(m, w, b, r, 1, lin=snap)
        assert r.counter == 256
        # shard-local gradient for those labels, (p - onehot)/256 on this shard's rows
        cot = lin.probs[rows].copy()
        cot[np.arange(128), labels[rows]] -= 1.0
        sub = O.linearize(dims, "relu", "ce", w.data, X[rows], y[rows])
        gh = O.vjp(sub, cot / 256)
        assert rel(est.data, 256 * gh * gh) < REL
    assert full.shape == est.data.shape


PRESETS = ["sophia_g", "sophia_h", "sophia_n", "adahessian", "adam", "sgdm", "sgd"]


@pytest.mark.parametrize("preset", PRESETS)
def test_preset_trajectory_matches_reference(golden, preset):
    """Four Method.step calls of the preset (device chain, estimator, diag lane) against
    the real reference's StepInfo rows and final weights."""
    g = golden("gnb_presets")
    m = P.Model(64, (96, 64), 10, "relu")
    w = P.init_params(m, P.Rng(0)).to_device()
    meth = P.make(preset, m)
    st = meth.init(w, 0)
    rows = []
    for t in range(4):
        X, y = O.synthetic_batch(128, 64, 10, seed=1 + t)
        w, st, info = meth.step(w, P.Batch(X, y, "ce"), st)
        rows.append(info.to_row())
    mine, ref = np.array(rows, dtype=np.float64), g[f"{preset}/info"]
    assert np.array_equal(np.isnan(mine), np.isnan(ref))
    ints = [P.STEP_INFO_FIELDS.index(f) for f in ("solver_iterations", "solver_converged", "step_index")]
    assert np.array_equal(mine[:, ints], ref[:, ints])
    ok = ~np.isnan(ref)
    np.testing.assert_allclose(mine[ok], ref[ok], rtol=REL, atol=1e-9)
    assert rel(w.data, g[f"{preset}/w_final"]) < 1e-5


def test_aborted_step_keeps_chain_state():
    """method.py:321-330: a non-finite batch returns the OLD chain state (momentum trace)."""
    m = P.Model(64, (96, 64), 10, "relu")
    w = P.init_params(m, P.Rng(0)).to_device()
    meth = P.make("sgdm", m)
    st = meth.init(w, 0)
    X, y = O.synthetic_batch(128, 64, 10)
    w1, st1, _ = meth.step(w, P.Batch(X, y, "ce"), st)
    trace = st1.chain[0]["trace"].clone()
    Xb = X.copy()
    Xb[0, 0] = np.inf
    w2, st2, info = meth.step(w1, P.Batch(Xb, y, "ce"), st1)
    assert info.solver_converged == -1 and info.step_norm == 0.0
    assert torch.equal(w2.data, w1.data)
    assert torch.equal(st2.chain[0]["trace"], trace)
