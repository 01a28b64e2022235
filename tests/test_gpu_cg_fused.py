"""The one-launch CG iteration (k_cg_fused, csrc/vec.cu) against the per-kernel
iteration (CURVOPT_CG_FUSED=0) across the per-thread register shares it is compiled
for (NQ = 1..4 groups of 16 bytes per thread), ragged tails (d % 4 = 1, 2, 3), with and
without the diagonal preconditioner, and with a stabilising iteration in the middle
(solvers.py:90-113): the same iteration counts and flags, iterates equal up to the
summation order and the split exponent (bound-derived vs exact amax: at most one bit
of the 22-bit split).

Seven iterations: on these b = 256 systems (GGN rank <= 2560, lam = 0.5) plain fp32 CG
starts amplifying rounding differences by the ninth iteration -- there the per-kernel path
is 6.7e-4 and the fused path 1.1e-4 from an f64 CG with the same masks
(scratch/cgf_oracle.py), so a fused-vs-per-kernel comparison there measures the
amplification, not the kernels."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (input, hidden, classes): d = 43 (d % 4 = 3, NQ 1), 269,322 (NQ 1), 669,706 (NQ 2),
# 1,575,937 (NQ 3, d % 4 = 1), 1,863,690 (NQ 4, the C3 model)
MODELS = [(4, (5,), 3), (784, (256, 256), 10), (784, (512, 512), 10), (512, (1024, 1024), 1),
          (784, (1024, 1024), 10)]

SCRIPT = r"""
import sys, json; sys.path.insert(0, %r)
import numpy as np, torch
import paper_2603_25976_b200 as P
from paper_2603_25976_b200.solvers import device_cg, read_cg_stats, CgConfig
out = []
for n0, hid, c in %r:
    m = P.Model(n0, hid, c, "relu")
    w = P.init_params(m, P.Rng(3)).to_device()
    r = P.Rng(5); b = 256
    X = torch.from_numpy(r.normal(b * n0).reshape(b, n0).astype(np.float32)).cuda()
    if c == 1:
        batch = P.Batch(X, torch.from_numpy(r.normal(b).reshape(b, 1).astype(np.float32)).cuda(), "mse")
        kind = "ggn_mse"
    else:
        batch = P.Batch(X, torch.from_numpy(r.integers(b, c)).cuda(), "ce")
        kind = "ggn_ce"
    snap = P.make_snapshot(kind, m, w, batch)
    g = snap.grad.data.clone()
    pre = torch.from_numpy(np.abs(r.normal(w.dim)).astype(np.float32)).cuda()
    for use_pre in (False, True):
        cfg = CgConfig(tol=1e-12, maxiter=7, stabilise_every=4)
        x, st = device_cg(snap, g, 0.5, cfg, precond=pre if use_pre else None)
        s = read_cg_stats(st)
        out.append({"d": w.dim, "pre": use_pre, "x": x.double().cpu().numpy().tolist(),
                    "it": s.iterations, "conv": s.converged, "neg": s.neg_curv, "gv": s.gv_count,
                    "relres": s.relres})
print(json.dumps(out))
""" % (ROOT, MODELS)


def _run(fused):
    env = dict(os.environ, CURVOPT_CG_FUSED=fused)
    p = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


def test_fused_iteration_matches_per_kernel_iteration_across_shapes():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    a, b = _run("0"), _run("1")
    assert len(a) == len(b) == 2 * len(MODELS)
    for ra, rb in zip(a, b):
        ctx = f"d={ra['d']} pre={ra['pre']}"
        assert (ra["it"], ra["conv"], ra["neg"], ra["gv"]) == (rb["it"], rb["conv"], rb["neg"], rb["gv"]), ctx
        xa, xb = np.array(ra["x"]), np.array(rb["x"])
        assert np.isfinite(xb).all(), ctx
        err = np.linalg.norm(xb - xa) / np.linalg.norm(xa)
        assert err <= 1e-5, (ctx, err)
        assert abs(rb["relres"] - ra["relres"]) <= 1e-3 * abs(ra["relres"]) + 1e-9, ctx
