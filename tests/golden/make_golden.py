"""Generate golden fixtures by running the REAL reference (`curvopt`).

Run in the build container only (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Outputs `tests/golden/*.npz` (committed).  Every case uses the reference's own
public API: `init_params`, `Rng`, `linearize`, `make_snapshot`, `cg_solve`,
`hutchinson_*`, `row_solve_cholesky`, `make(...)` + `Method.step`.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("CURVOPT_REF", "/root/reference/pkg/src"))

from curvopt import numeric as N  # noqa: E402
from curvopt.curvature import make_snapshot  # noqa: E402
from curvopt.harness.data import gen_classification  # noqa: E402
from curvopt.harness.run import EpochBatcher  # noqa: E402
from curvopt.method import (  # noqa: E402
    CurvatureSpec, DampingSpec, EstimatorSpec, MethodSpec, PrecondSpec, SolverSpec,
    TelemetrySpec, assemble,
)
from curvopt.models import Batch, Model, init_params, linearize  # noqa: E402
from curvopt.control import TrustRegionConfig  # noqa: E402
from curvopt.solvers import CgConfig, cg_solve, row_solve_cholesky  # noqa: E402
from curvopt.telemetry import hutchinson_diag, hutchinson_trace, power_iter_top_eig  # noqa: E402
from curvopt.transforms import (add_decayed_weights, chain_apply, chain_init, clip_global_norm,  # noqa: E402
                                scale, scale_by_adam, scale_by_schedule, sophia_clip, trace_momentum)


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print("wrote", path, sum(a.nbytes for a in map(np.asarray, arrays.values())), "bytes")


def rng_cases():
    out = {}
    cases = [(0, 0, 1000), (42, 101770, 5000), (2**64 - 1, 7, 100), (123456789, 0, 4096)]
    for i, (s, c, n) in enumerate(cases):
        r = N.Rng(s, c)
        out[f"raw{i}"] = r._raw(n)
        out[f"rad{i}"] = N.rademacher(N.Rng(s, c), n)
        out[f"uni{i}"] = N.Rng(s, c).uniform(n)
        out[f"nrm{i}"] = N.Rng(s, c).normal(n + 1)  # odd count exercises the tail
        out[f"int{i}"] = N.Rng(s, c).integers(n, 10)
        out[f"perm{i}"] = N.Rng(s, c).permutation(min(n, 500))
        child = N.Rng(s, c).split()
        out[f"split{i}"] = np.array([child.seed], dtype=np.uint64)
        out[f"case{i}"] = np.array([s, c, n], dtype=np.uint64)
    save("rng", **out)


def batch_for(model, b, loss, seed=1):
    r = N.Rng(seed)
    X = r.normal(b * model.input_dim).reshape(b, model.input_dim)
    y = r.integers(b, model.output_dim) if loss == "ce" else r.normal(b * model.output_dim).reshape(b, model.output_dim)
    return Batch(X, y, loss)


def primitive_cases():
    """Small nets: every hot-path primitive at identical inputs."""
    out = {}
    cfgs = [
        ("relu_ce", Model(12, (16, 8), 5, "relu"), "ce", 9),
        ("tanh_ce", Model(12, (16, 8), 5, "tanh"), "ce", 9),
        ("relu_mse", Model(12, (16, 8), 3, "relu"), "mse", 7),
        ("tanh_mse", Model(6, (10,), 2, "tanh"), "mse", 5),
        ("lin_ce", Model(6, (), 4, "relu"), "ce", 6),
    ]
    for name, m, loss, b in cfgs:
        w = init_params(m, N.Rng(0))
        batch = batch_for(m, b, loss)
        lin = linearize(m, w, batch)
        d = w.dim
        v = w.like(N.Rng(2).normal(d))
        U = N.Rng(3).normal(b * m.output_dim).reshape(b, m.output_dim)
        kind = "ggn_ce" if loss == "ce" else "ggn_mse"
        snap = make_snapshot(kind, m, w, batch)
        hsnap = make_snapshot("hessian", m, w, batch)
        cfg = CgConfig(tol=1e-5, maxiter=10, stabilise_every=3, warm_start=True)
        res = cg_solve(snap.matvec, snap.grad, 0.5, cfg)
        pre = w.like(np.abs(N.Rng(4).normal(d)))
        res_p = cg_solve(snap.matvec, snap.grad, 0.5, cfg, precond=pre, x0=w.like(N.Rng(6).normal(d) * 1e-2))
        mv = lambda x: snap.matvec(w.like(x)).data  # noqa: E731
        rng = N.Rng(5)
        hd = hutchinson_diag(mv, rng, d, 3)
        ht = hutchinson_trace(mv, rng, d, 2)
        pe = power_iter_top_eig(mv, rng, d, 7)
        gram = snap.row.gram()
        mu = float(b) * 0.7
        vrow = row_solve_cholesky(gram, snap.row.rhs, mu)
        rowdir = snap.row.scaled_row_transpose(vrow).data
        seeds = lin.hz_half()
        out.update({
            f"{name}/dims": np.array(m.dims), f"{name}/act": np.array(m.activation),
            f"{name}/loss": np.array(loss), f"{name}/w": w.data, f"{name}/X": batch.inputs,
            f"{name}/y": batch.targets, f"{name}/v": v.data, f"{name}/U": U,
            f"{name}/value": np.array(lin.loss), f"{name}/grad": lin.grad.data,
            f"{name}/out": lin.out, f"{name}/jvp": lin.jvp(v), f"{name}/vjp": lin.vjp(U).data,
            f"{name}/ggn": snap.matvec(v).data, f"{name}/hvp": hsnap.matvec(v).data,
            f"{name}/cg_x": res.direction.data,
            f"{name}/cg_stats": np.array([res.iterations, res.converged, res.final_relative_residual, res.negative_curvature], dtype=np.float64),
            f"{name}/pcg_pre": pre.data, f"{name}/pcg_x0": N.Rng(6).normal(d) * 1e-2,
            f"{name}/pcg_x": res_p.direction.data,
            f"{name}/pcg_stats": np.array([res_p.iterations, res_p.converged, res_p.final_relative_residual, res_p.negative_curvature], dtype=np.float64),
            f"{name}/hutch_diag": hd, f"{name}/hutch_trace": np.array(ht), f"{name}/top_eig": np.array(pe),
            f"{name}/rng_after": np.array([rng.counter], dtype=np.int64),
            f"{name}/seeds": seeds, f"{name}/rhs": snap.row.rhs, f"{name}/gram": gram,
            f"{name}/mu": np.array(mu), f"{name}/rowdir": rowdir,
            f"{name}/loss_at": np.array(snap.loss_at(w.like(w.data + 0.01 * v.data))),
        })
    save("primitives", **out)


def _spec(**kw):
    cg = CgConfig(tol=1e-5, maxiter=kw.pop("maxiter", 10), stabilise_every=10, warm_start=True)
    return MethodSpec(
        curvature=CurvatureSpec(kw.pop("curvature", "ggn_ce")),
        solver=SolverSpec(kw.pop("solver", "cg"), cg),
        precond=kw.pop("precond", None),
        damping=kw.pop("damping", DampingSpec("constant", 1.0)),
        estimator=kw.pop("estimator", None),
        telemetry=kw.pop("telemetry", TelemetrySpec()),
        chain=(scale(1e-3), scale(-1.0)),
    )


def run_steps(spec, model, w, batches, seed=0):
    meth = assemble(spec, model)
    st = meth.init(w, seed)
    rows = []
    for batch in batches:
        w, st, info = meth.step(w, batch, st)
        rows.append(info.to_row())
    return np.array(rows, dtype=np.float64), w.data


def trajectory_cases():
    out = {}
    # C1: 784-128-10 CE b=128, GGN + CG(10) + constant lam=1, one step (+ a second on the same batch)
    m1 = Model(784, (128,), 10, "relu")
    w1 = init_params(m1, N.Rng(0))
    b1 = batch_for(m1, 128, "ce")
    meth = assemble(_spec(), m1)
    st = meth.init(w1, 0)
    lin = linearize(m1, w1, b1)
    wn, st, info = meth.step(w1, b1, st)
    out["c1/info0"] = np.array(info.to_row(), dtype=np.float64)
    out["c1/grad"] = lin.grad.data.astype(np.float32)
    out["c1/direction"] = st.warm_start.astype(np.float32)
    wn2, st, info = meth.step(wn, b1, st)
    out["c1/info1"] = np.array(info.to_row(), dtype=np.float64)
    out["c1/w2_norm"] = np.array(np.linalg.norm(wn2.data))

    # C2: C1 + trust region (every 5) + Hutchinson@10, 100 steps on gen_classification batches
    train, _ = gen_classification(20000, 784, 10, 10.0, 0)
    batcher = EpochBatcher(train, 128, N.Rng(0).split())
    batches = [batcher.next() for _ in range(100)]
    spec2 = _spec(damping=DampingSpec("trust_region", 1.0, TrustRegionConfig(every_k=5)),
                  estimator=EstimatorSpec("hutchinson", 1, every_k=10))
    rows, wf = run_steps(spec2, m1, w1, batches)
    out["c2/info"] = rows
    out["c2/w_final_norm"] = np.array(np.linalg.norm(wf))
    out["c2/first_batch_idx_sum"] = np.array(float(batches[0].inputs.sum()))

    # C3-shaped, reduced batch: 784-1024-1024-10, b=256, PCG fed by diag-EMA(0.99) + Hutchinson@2
    m3 = Model(784, (1024, 1024), 10, "relu")
    w3 = init_params(m3, N.Rng(0))
    b3 = batch_for(m3, 256, "ce")
    spec3 = _spec(precond=PrecondSpec("diag_ema", 0.99), estimator=EstimatorSpec("hutchinson", 1, every_k=2))
    rows, wf = run_steps(spec3, m3, w3, [b3] * 3)
    out["c3r/info"] = rows
    out["c3r/w_final_norm"] = np.array(np.linalg.norm(wf))

    # C4-shaped, reduced: row-space Cholesky lane, 96-64-64-10 CE b=32
    m4 = Model(96, (64, 64), 10, "relu")
    w4 = init_params(m4, N.Rng(0))
    b4 = batch_for(m4, 32, "ce")
    rows, wf = run_steps(_spec(solver="row_cholesky"), m4, w4, [b4] * 2)
    out["c4r/info"] = rows
    out["c4r/w_final"] = wf

    # C5-shaped, reduced: exact Hessian + CG, constant damping, trace + Hutchinson telemetry
    m5 = Model(48, (32, 32, 32, 32), 10, "relu")
    w5 = init_params(m5, N.Rng(0))
    b5 = batch_for(m5, 64, "ce")
    spec5 = _spec(curvature="hessian", estimator=EstimatorSpec("hutchinson", 1, every_k=1),
                  telemetry=TelemetrySpec(trace_every_k=1, trace_probes=2, rho_every_k=2))
    rows, wf = run_steps(spec5, m5, w5, [b5] * 3)
    out["c5r/info"] = rows
    out["c5r/w_final"] = wf
    save("trajectories", **out)


def plan_cases():
    """Plans of every preset and the stable AssemblyError messages (method.py:181-218, 412-552)."""
    import dataclasses
    import json

    from curvopt.errors import AssemblyError
    from curvopt.method import PRESET_NAMES, make

    m = Model(6, (5,), 3, "relu")
    plans = {}
    for name in PRESET_NAMES:
        p = make(name, m).plan
        g = p.gates
        plans[name] = {
            "lane": p.lane, "algo": p.algo, "schema": list(p.schema),
            "gates": {k: getattr(g, k).k for k in ("rho", "trace", "top_eig", "estimator", "tr_rho")},
            "solver_config": dataclasses.asdict(p.solver_config),
            "needs_row_primitives": p.needs_row_primitives, "needs_rho": p.needs_rho,
        }
    bad = {
        "solver_without_curvature": {"curvature": None},
        "row_with_hessian": {"curvature": {"kind": "hessian"}, "solver": {"kind": "row_cholesky"}},
        "diag_without_source": {"solver": {"kind": "diag"}},
        "gnb_with_mse": {"curvature": {"kind": "ggn_mse"}, "estimator": {"kind": "gnb"}},
        "sq_grad_with_estimator": {"precond": {"kind": "sq_grad"}, "estimator": {"kind": "hutchinson"}},
        "ema_without_estimator": {"precond": {"kind": "diag_ema"}},
        "tr_disabled_cadence": {"damping": {"policy": "trust_region", "tr": {"every_k": -1}}},
        "unknown_field": {"bogus": 1},
        "unknown_curvature": {"curvature": {"kind": "fisher"}},
        "unknown_solver": {"solver": {"kind": "lbfgs"}},
        "unknown_policy": {"damping": {"policy": "step_norm"}},
    }
    msgs = {}
    for key, ov in bad.items():
        try:
            make("sgn_ce", m, **ov)
            msgs[key] = None
        except (AssemblyError, TypeError, ValueError) as e:
            msgs[key] = f"{type(e).__name__}: {e}"
    for key, ov in {"telemetry_without_curvature": {"telemetry": {"rho_every_k": 2}},
                    "tr_without_curvature": {"damping": {"policy": "trust_region"}}}.items():
        try:
            make("sgd", m, **ov)
            msgs[key] = None
        except (AssemblyError, ValueError) as e:
            msgs[key] = f"{type(e).__name__}: {e}"
    with open(os.path.join(HERE, "plans.json"), "w") as f:
        json.dump({"plans": plans, "errors": msgs, "overrides": {k: v for k, v in bad.items()}}, f, indent=1,
                  sort_keys=True)
    print("wrote plans.json")


def primitive_tc_cases():
    """Batch >= 128 and widths >= 64: every GEMM of the linearization, the GGN product and
    the HVP runs on the tensor-core engine (M >= 64, 16-byte rows), and the output layer
    takes the transposed tensor-core path (c >= 8, b >= 128)."""
    out = {}
    cfgs = [
        ("relu_ce", Model(64, (96, 64), 10, "relu"), "ce", 128),
        ("tanh_ce", Model(64, (96, 64), 10, "tanh"), "ce", 128),
        ("relu_mse", Model(64, (128,), 8, "relu"), "mse", 192),
        ("tanh_mse", Model(64, (64, 64), 8, "tanh"), "mse", 128),
    ]
    for name, m, loss, b in cfgs:
        w = init_params(m, N.Rng(0))
        batch = batch_for(m, b, loss)
        lin = linearize(m, w, batch)
        d = w.dim
        v = w.like(N.Rng(2).normal(d))
        U = N.Rng(3).normal(b * m.output_dim).reshape(b, m.output_dim)
        kind = "ggn_ce" if loss == "ce" else "ggn_mse"
        snap = make_snapshot(kind, m, w, batch)
        hsnap = make_snapshot("hessian", m, w, batch)
        cfg = CgConfig(tol=1e-5, maxiter=10, stabilise_every=3, warm_start=True)
        res = cg_solve(snap.matvec, snap.grad, 0.5, cfg)
        hres = cg_solve(hsnap.matvec, snap.grad, 2.0, cfg)
        mv = lambda x: snap.matvec(w.like(x)).data  # noqa: E731
        rng = N.Rng(5)
        hd = hutchinson_diag(mv, rng, d, 2)
        ht = hutchinson_trace(mv, rng, d, 2)
        out.update({
            f"{name}/dims": np.array(m.dims), f"{name}/act": np.array(m.activation),
            f"{name}/loss": np.array(loss), f"{name}/w": w.data, f"{name}/X": batch.inputs,
            f"{name}/y": batch.targets, f"{name}/v": v.data, f"{name}/U": U,
            f"{name}/value": np.array(lin.loss), f"{name}/grad": lin.grad.data,
            f"{name}/out": lin.out, f"{name}/jvp": lin.jvp(v), f"{name}/vjp": lin.vjp(U).data,
            f"{name}/ggn": snap.matvec(v).data, f"{name}/hvp": hsnap.matvec(v).data,
            f"{name}/cg_x": res.direction.data,
            f"{name}/cg_stats": np.array([res.iterations, res.converged, res.final_relative_residual], dtype=np.float64),
            f"{name}/hcg_x": hres.direction.data,
            f"{name}/hcg_stats": np.array([hres.iterations, hres.converged, hres.final_relative_residual,
                                           hres.negative_curvature], dtype=np.float64),
            f"{name}/hutch_diag": hd, f"{name}/hutch_trace": np.array(ht),
            f"{name}/loss_at": np.array(snap.loss_at(w.like(w.data + 0.01 * v.data))),
        })
    save("primitives_tc", **out)


CHAINS = {
    "sophia": lambda: (trace_momentum(0.96), sophia_clip(0.05, 1e-12), add_decayed_weights(1e-4),
                       scale_by_schedule("constant", alpha0=0.01), scale(-1.0)),
    "adam": lambda: (scale_by_adam(0.9, 0.999, 1e-8), scale_by_schedule("constant", alpha0=1e-3), scale(-1.0)),
    "sgdm": lambda: (trace_momentum(0.9), add_decayed_weights(5e-4), scale_by_schedule("constant", alpha0=0.05),
                     scale(-1.0)),
    "clip_cos": lambda: (clip_global_norm(0.5), scale_by_schedule("cosine_warmup", alpha0=0.3, warmup=2, total=6),
                         trace_momentum(0.5), clip_global_norm(0.05), scale(-2.0)),
    "step_decay": lambda: (scale_by_schedule("step_decay", alpha0=0.2, gamma=0.5, period=2), scale(-1.0)),
}


def chain_cases():
    """The reference's transform chains (transforms.py:148-199) over 4 steps of random
    directions: update and the threaded state per step."""
    out = {}
    d = 3001
    lay = (("w", (d,)),)
    for name, mk in CHAINS.items():
        chain = mk()
        w = N.ParamVector(N.Rng(11).normal(d), lay)
        pre = N.ParamVector(np.abs(N.Rng(12).normal(d)) * 1e-2, lay)
        st = chain_init(chain, w)
        for t in range(4):
            direc = N.ParamVector(N.Rng(20 + t).normal(d) * (3.0 if t == 1 else 1.0), lay)
            upd, st = chain_apply(chain, st, direc, w, t, precond_diag=pre)
            out[f"{name}/upd{t}"] = upd.data
            for i, s in enumerate(st):
                for key, val in s.items():
                    out[f"{name}/st{t}_{i}_{key}"] = np.asarray(val, dtype=np.float64)
            w = w + upd
        out[f"{name}/w0"] = N.Rng(11).normal(d)
        out[f"{name}/pre"] = pre.data
    save("chains", **out)


def gnb_cases():
    """Sampled-label GNB diagonal (telemetry.py:129-160) and the Sophia-G / AdaHessian /
    Adam / SGDM presets over a few steps (device transform chains through Method.step)."""
    from curvopt.method import make
    from curvopt.telemetry import gnb_diag

    out = {}
    m = Model(64, (96, 64), 10, "relu")
    w = init_params(m, N.Rng(0))
    batch = batch_for(m, 128, "ce")
    rng = N.Rng(7)
    out["gnb/diag"] = gnb_diag(m, w, batch, rng, 3).data
    out["gnb/rng_after"] = np.array([rng.counter], dtype=np.int64)
    for preset in ("sophia_g", "sophia_h", "sophia_n", "adahessian", "adam", "sgdm", "sgd"):
        meth = make(preset, m)
        st = meth.init(w, 0)
        ww = w
        rows = []
        for t in range(4):
            ww, st, info = meth.step(ww, batch_for(m, 128, "ce", seed=1 + t), st)
            rows.append(info.to_row())
        out[f"{preset}/info"] = np.array(rows, dtype=np.float64)
        out[f"{preset}/w_final"] = ww.data
    save("gnb_presets", **out)


def harness_cases():
    """Synthetic regression + epoch batches of the cadence study (data.py:49-60,
    run.py:174-192, bench.py:135-207): first batches and a short newton_cg run."""
    from curvopt.harness.data import gen_regression
    from curvopt.method import make

    out = {}
    train, test = gen_regression(n=2000, d=32, noise_std=0.1, seed=0)
    out["reg/train_X_sum"] = np.array(train.X.sum())
    out["reg/train_y"] = train.y[:50, 0].copy()
    out["reg/test_n"] = np.array(test.n)
    root = N.Rng(0)
    m = Model(32, (64, 64), 1, "relu")
    w = init_params(m, root.split())
    batcher = EpochBatcher(train, 128, root.split())
    meth = make("newton_cg", m, damping={"policy": "constant", "lam0": 1.0, "tr": None},
                solver={"cg": {"maxiter": 3, "warm_start": True}}, telemetry={"rho_every_k": 2})
    st = meth.init(w, seed=0)
    rows = []
    for t in range(6):
        b = batcher.next()
        if t == 0:
            out["reg/batch0_idx_X"] = b.inputs[:4].copy()
        w, st, info = meth.step(w, b, st)
        rows.append(info.to_row())
    out["newton_cg/info"] = np.array(rows, dtype=np.float64)
    out["newton_cg/w_final"] = w.data
    save("harness", **out)


def rowcg_cases():
    """The row-space CG lane (egn_mse_cg: method.py:270-282, solvers.py:164-174) over a
    few steps of the lane-scaling workload (bench.py:67-82), warm-started from the
    previous row-space solution; plus one row_solve_cg on a snapshot Gram."""
    from curvopt.harness.data import gen_regression
    from curvopt.method import make
    from curvopt.solvers import row_solve_cg

    out = {}
    train, _ = gen_regression(n=2000, d=32, noise_std=0.1, seed=0)
    root = N.Rng(0)
    m = Model(32, (64, 64), 1, "relu")
    w = init_params(m, root.split())
    batcher = EpochBatcher(train, 96, root.split())
    meth = make("egn_mse_cg", m)
    st = meth.init(w, seed=0)
    rows = []
    for t in range(5):
        b = batcher.next()
        if t == 0:
            snap = make_snapshot("ggn_mse", m, w, b)
            gram = snap.row.gram()
            v, it, conv, rr = row_solve_cg(lambda u: gram @ u, snap.row.rhs, 96.0,
                                           CgConfig(tol=1e-5, maxiter=10, stabilise_every=10, warm_start=True))
            out["solve/v"] = v
            out["solve/stats"] = np.array([it, int(conv), rr])
        w, st, info = meth.step(w, b, st)
        rows.append(info.to_row())
    out["egn_mse_cg/info"] = np.array(rows, dtype=np.float64)
    out["egn_mse_cg/w_final"] = w.data
    save("rowcg", **out)


if __name__ == "__main__":
    rng_cases()
    primitive_cases()
    trajectory_cases()
    plan_cases()
    primitive_tc_cases()
    chain_cases()
    gnb_cases()
    harness_cases()
    rowcg_cases()
