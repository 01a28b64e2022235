"""CPU tests of the host mirror of the reference API: plan output bit-exact
with the reference (golden plans.json from the real reference), stable
assembly-error messages, StepInfo schema / sentinels, cadence law, RNG and
initialisation bit-exactness, transforms on host arrays."""

import json
import math
import os

import numpy as np
import pytest

import paper_2603_25976_b200 as P
from paper_2603_25976_b200.errors import AssemblyError, ContractError

GOLD = os.path.join(os.path.dirname(__file__), "golden", "plans.json")
M = P.Model(6, (5,), 3, "relu")


def _plan_dict(p):
    import dataclasses

    g = p.gates
    return {"lane": p.lane, "algo": p.algo, "schema": list(p.schema),
            "gates": {k: getattr(g, k).k for k in ("rho", "trace", "top_eig", "estimator", "tr_rho")},
            "solver_config": dataclasses.asdict(p.solver_config),
            "needs_row_primitives": p.needs_row_primitives, "needs_rho": p.needs_rho}


def test_presets_and_plans_bit_exact():
    gold = json.load(open(GOLD))
    assert tuple(gold["plans"]) == P.PRESET_NAMES or set(gold["plans"]) == set(P.PRESET_NAMES)
    for name, ref in gold["plans"].items():
        assert _plan_dict(P.make(name, M).plan) == ref, name


def test_assembly_error_messages_stable():
    gold = json.load(open(GOLD))
    overrides = gold["overrides"]
    for key, msg in gold["errors"].items():
        if key in overrides:
            base, ov = "sgn_ce", overrides[key]
        elif key == "telemetry_without_curvature":
            base, ov = "sgd", {"telemetry": {"rho_every_k": 2}}
        else:
            base, ov = "sgd", {"damping": {"policy": "trust_region"}}
        with pytest.raises(AssemblyError) as ei:
            P.make(base, M, **ov)
        assert f"AssemblyError: {ei.value}" == msg


def test_step_info_schema_and_sentinels():
    assert P.STEP_INFO_FIELDS == ("loss_before", "loss_after", "rho", "lam", "grad_norm", "step_norm",
                                  "solver_iterations", "solver_converged", "final_relative_residual",
                                  "diag_mean", "trace_estimate", "top_eig_estimate", "step_index")
    info = P.StepInfo()
    row = info.to_row()
    assert len(row) == 13 and math.isnan(row[0]) and row[6] == -1 and row[12] == -1
    plan = P.make("sgn_ce", M).plan
    packed = P.pack_step_info(plan, {"solver_iterations": 3.0, "lam": 2})
    assert packed.solver_iterations == 3 and isinstance(packed.solver_iterations, int) and packed.lam == 2.0
    with pytest.raises(ContractError):
        P.pack_step_info(plan, {"bogus": 1})


def test_cadence_law():
    c = P.Cadence(5)
    assert [t for t in range(12) if c.fires(t)] == [0, 5, 10]
    assert not any(P.Cadence(-1).fires(t) for t in range(10))
    with pytest.raises(ContractError):
        P.Cadence(0)


def test_rng_and_init_bit_exact(golden):
    g = golden("rng")
    for i in range(4):
        s, c, n = (int(x) for x in g[f"case{i}"])
        assert np.array_equal(P.Rng(s, c)._raw(n), g[f"raw{i}"])
        assert np.array_equal(P.rademacher(P.Rng(s, c), n), g[f"rad{i}"])
        assert np.array_equal(P.Rng(s, c).normal(n + 1), g[f"nrm{i}"])
        assert np.array_equal(P.Rng(s, c).permutation(min(n, 500)), g[f"perm{i}"])
        assert P.Rng(s, c).split().seed == int(g[f"split{i}"][0])
    p = golden("primitives")
    dims = tuple(int(x) for x in p["relu_ce/dims"])
    m = P.Model(dims[0], dims[1:-1], dims[-1], "relu")
    assert np.array_equal(P.init_params(m, P.Rng(0)).data, p["relu_ce/w"])


def test_overrides_and_module_diff():
    spec = P.preset_spec("sgn_mse", solver={"cg": {"maxiter": 3}})
    assert spec.solver.cg.maxiter == 3 and spec.solver.cg.tol == 1e-5
    spec = P.preset_spec("sgn_mse", damping={"policy": "trust_region", "tr": {"every_k": 2}})
    assert spec.damping.tr.every_k == 2
    assert P.module_diff(P.preset_spec("sophia_n"), P.preset_spec("sophia_g")) == ("estimator",)
    assert P.module_diff(P.preset_spec("sophia_n"), P.preset_spec("sophia_h")) == ("curvature",)


@pytest.mark.gpu
def test_chain_apply_host_arrays():
    """Host ParamVectors go through the device chain kernel (no CPU path)."""
    w = P.ParamVector(np.arange(4.0), (("w", (4,)),))
    d = w.like(np.ones(4))
    chain = (P.transforms.trace_momentum(0.5), P.transforms.clip_global_norm(1.0), P.transforms.scale(-2.0))
    st = P.chain_init(chain, w)
    u, st = P.chain_apply(chain, st, d, w, 0)
    np.testing.assert_allclose(u.data, -2.0 * np.ones(4) / 2.0)
    u, st = P.chain_apply(chain, st, d, w, 1)  # momentum 1.5, clipped to norm 1
    np.testing.assert_allclose(np.linalg.norm(u.data), 2.0)
    assert P.schedule_value("cosine_warmup", 5, {"alpha0": 1.0, "warmup": 10, "total": 20}) == 0.5


def test_param_vector_contracts():
    lay = P.models.param_layout(M)
    with pytest.raises(ContractError):
        P.ParamVector(np.zeros(3), lay)
    a = P.ParamVector(np.zeros(P.models.param_count(M)), lay)
    with pytest.raises(ContractError):
        a + P.ParamVector(np.zeros(3), (("x", (3,)),))
    with pytest.raises(ContractError):
        P.Batch(np.zeros((2, 6)), np.array([0.5, 1.5]), "ce")


def test_damping_and_rho_rules():
    from paper_2603_25976_b200.control import DampingState, RhoBundle, damping_update, escalate_damping, rho_from_terms

    st = DampingState(1.0, "trust_region")
    assert damping_update(st, RhoBundle(0, 0, 1, 0.9), 0).lam == 0.5
    assert damping_update(st, RhoBundle(0, 0, 1, 0.1), 0).lam == 1.5
    assert damping_update(st, RhoBundle(0, 0, 1, float("nan")), 0).lam == 1.0
    assert escalate_damping(st).lam == 1.5
    assert math.isnan(rho_from_terms(1.0, 0.5, 1.0, 1.0).rho)  # pred <= 0
    assert rho_from_terms(1.0, 0.0, -1.0, 0.0).rho == 1.0
    assert rho_from_terms(10.0, -100.0, -1.0, 0.0).rho == 5.0  # clipped


def test_batch_label_range_hint_from_host_labels():
    """A loader holding the host copy of the labels passes their min/max (no device read);
    a negative minimum is still the reference's contract error (models.py Batch)."""
    import torch

    from paper_2603_25976_b200 import Batch
    from paper_2603_25976_b200.errors import ContractError

    X = torch.zeros(4, 3)
    y = torch.tensor([0, 2, 1, 2])
    b = Batch(X, y, "ce", _dev={"_ymin": 0, "_ymax": 2})
    assert b.max_label() == 2
    with pytest.raises(ContractError):
        Batch(X, y, "ce", _dev={"_ymin": -1, "_ymax": 2})
    with pytest.raises(ContractError):
        Batch(X, torch.tensor([0, -1, 1, 2]), "ce")
