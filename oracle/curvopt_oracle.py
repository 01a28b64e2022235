"""CPU oracle for the curvature-matvec hot path -- TEST INFRASTRUCTURE ONLY.

This module is a float64 numpy restatement of the reference package
`curvopt` 0.1.0 (paths below are relative to /root/reference/pkg/src/curvopt).
It exists so that the GPU path can be checked on the GPU box, where the
reference itself is not available.  Only `tests/`, `__graft_entry__.smoke()` and
the `cpu_baseline` / `--impl reference` legs of `bench.py` may import it; the
product package (`paper_2603_25976_b200`) never does.

Parity status: PINNED.  `tests/golden/make_golden.py` runs the real reference
(importable in the build container) and stores fixtures under `tests/golden/`;
`tests/test_oracle_golden.py` checks this restatement against every one of them
(RNG streams bit-exact, numerics to 1e-12 relative).

The structure is deliberately functional (a `Lin` record + free functions)
rather than the reference's class layout; each function names the reference
lines whose behaviour it restates.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

U64 = np.uint64
MASK64 = (1 << 64) - 1

# --------------------------------------------------------------------------
# SplitMix64 counter stream  (numeric.py:95-162)
# --------------------------------------------------------------------------
_G = U64(0x9E3779B97F4A7C15)
_M1 = U64(0xBF58476D1CE4E5B9)
_M2 = U64(0x94D049BB133111EB)


def splitmix_block(seed: int, counter: int, n: int) -> np.ndarray:
    """Outputs for indices counter+1 .. counter+n (numeric.py:101-104, 124-128)."""
    idx = np.arange(counter + 1, counter + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = U64(seed & MASK64) + _G * idx
        x = (x ^ (x >> U64(30))) * _M1
        x = (x ^ (x >> U64(27))) * _M2
        return x ^ (x >> U64(31))


class ORng:
    """Counter RNG with the reference's draw semantics (numeric.py:107-154)."""

    def __init__(self, seed: int, counter: int = 0):
        self.seed = int(seed) & MASK64
        self.counter = int(counter)

    def clone(self) -> "ORng":
        return ORng(self.seed, self.counter)

    def raw(self, n: int) -> np.ndarray:
        out = splitmix_block(self.seed, self.counter, n)
        self.counter += n
        return out

    def uniform(self, n):  # numeric.py:130-132
        return (self.raw(n) >> U64(11)).astype(np.float64) * 2.0**-53

    def normal(self, n):  # numeric.py:134-142 (Box-Muller, first half cos, second sin)
        h = (n + 1) // 2
        u = self.raw(2 * h)
        a = ((u[:h] >> U64(11)).astype(np.float64) + 0.5) * 2.0**-53
        t = (u[h:] >> U64(11)).astype(np.float64) * 2.0**-53
        rad = np.sqrt(-2.0 * np.log(a))
        ang = 2 * np.pi * t
        return np.concatenate([rad * np.cos(ang), rad * np.sin(ang)])[:n]

    def integers(self, n, bound):  # numeric.py:144-146
        return np.minimum((self.uniform(n) * bound).astype(np.int64), bound - 1)

    def permutation(self, n):  # numeric.py:148-149
        return np.argsort(self.uniform(n), kind="stable")

    def split(self) -> "ORng":  # numeric.py:151-154
        return ORng(int(self.raw(1)[0]), 0)


def rademacher(rng: ORng, n: int) -> np.ndarray:
    """+-1 from the top bit of each draw (numeric.py:157-162)."""
    return (rng.raw(n) >> U64(63)).astype(np.float64) * 2.0 - 1.0


# --------------------------------------------------------------------------
# Flat parameter layout  (models.py:87-140)
# --------------------------------------------------------------------------

def n_params(dims) -> int:
    return sum((dims[i] + 1) * dims[i + 1] for i in range(len(dims) - 1))


def split_params(dims, flat):
    """Per layer (W[in,out] row-major, b[out]) views of the flat vector (models.py:115-128)."""
    out, off = [], 0
    for i in range(len(dims) - 1):
        fi, fo = dims[i], dims[i + 1]
        W = flat[off:off + fi * fo].reshape(fi, fo)
        off += fi * fo
        out.append((W, flat[off:off + fo]))
        off += fo
    return out


def join_params(parts) -> np.ndarray:
    """Inverse of split_params (models.py:131-140)."""
    return np.concatenate([np.concatenate([W.ravel(), b.ravel()]) for W, b in parts])


def init_params(dims, activation, rng: ORng) -> np.ndarray:
    """Gaussian init, gain sqrt(2) on relu hidden layers, zero bias (models.py:101-112)."""
    L = len(dims) - 1
    chunks = []
    for i in range(L):
        gain = math.sqrt(2.0) if (i < L - 1 and activation == "relu") else 1.0
        chunks.append(rng.normal(dims[i] * dims[i + 1]) * (gain / math.sqrt(dims[i])))
        chunks.append(np.zeros(dims[i + 1]))
    return np.concatenate(chunks)


# --------------------------------------------------------------------------
# Linearization  (models.py:165-396)
# --------------------------------------------------------------------------

@dataclass
class Lin:
    dims: tuple
    activation: str
    loss: str               # "mse" | "ce"
    X: np.ndarray
    y: np.ndarray
    layers: list            # [(W, b)]
    acts: list              # acts[l] = input of layer l
    sp: list                # activation derivative per hidden layer
    out: np.ndarray
    value: float            # batch mean loss
    out_grad: np.ndarray    # per-example dl/dz (no 1/b)
    G: list                 # dL/dz_l of the mean loss
    grad: np.ndarray
    probs: np.ndarray | None = None
    roots: tuple | None = field(default=None, repr=False)

    @property
    def b(self) -> int:
        return self.X.shape[0]

    @property
    def L(self) -> int:
        return len(self.layers)


def _ce_value(out, y):
    """Mean softmax-CE with max shift (models.py:367-370, 405-408)."""
    s = out - out.max(axis=1, keepdims=True)
    lse = np.log(np.exp(s).sum(axis=1))
    return float(np.mean(lse - s[np.arange(out.shape[0]), y]))


def _act(z, activation):
    return np.maximum(z, 0.0) if activation == "relu" else np.tanh(z)


def forward(dims, activation, flat, X) -> np.ndarray:
    """Network outputs (models.py:143-156)."""
    a = np.asarray(X, dtype=np.float64)
    layers = split_params(dims, flat)
    for i, (W, bias) in enumerate(layers):
        z = a @ W + bias
        a = _act(z, activation) if i < len(layers) - 1 else z
    return a


def loss_value(dims, activation, loss, flat, X, y) -> float:
    """Loss only, forward pass (models.py:399-408)."""
    out = forward(dims, activation, flat, X)
    if loss == "mse":
        r = out - np.asarray(y, dtype=np.float64).reshape(out.shape)
        return 0.5 * float(np.sum(r * r)) / out.shape[0]
    return _ce_value(out, y)


def linearize(dims, activation, loss, flat, X, y, masks=None) -> Lin:
    """Forward, loss, primal backward and gradient (models.py:337-396).

    `masks` (relu only, test instrumentation): per hidden layer the boolean
    "z > 0" pattern to use instead of the oracle's own -- the "identical inputs"
    override that removes fp32-vs-f64 ReLU kink flips from a parity comparison
    (hard part 2)."""
    X = np.asarray(X, dtype=np.float64)
    layers = split_params(dims, np.asarray(flat, dtype=np.float64))
    L = len(layers)
    acts, sp = [X], []
    a = X
    for i, (W, bias) in enumerate(layers):
        z = a @ W + bias
        if i == L - 1:
            out = z
            break
        if activation == "relu":
            keep = (z > 0.0) if masks is None else np.asarray(masks[i], dtype=bool)
            a = np.where(keep, z, 0.0)
            sp.append(keep.astype(np.float64))
        else:
            a = np.tanh(z)
            sp.append(1.0 - a * a)
        acts.append(a)
    b = X.shape[0]
    probs = None
    if loss == "mse":
        y = np.asarray(y, dtype=np.float64).reshape(out.shape)
        r = out - y
        value = 0.5 * float(np.sum(r * r)) / b
        og = r
    else:
        y = np.asarray(y, dtype=np.int64)
        value = _ce_value(out, y)
        e = np.exp(out - out.max(axis=1, keepdims=True))
        probs = e / e.sum(axis=1, keepdims=True)
        og = probs.copy()
        og[np.arange(b), y] -= 1.0
    G = [None] * L
    G[L - 1] = og / b
    for i in range(L - 1, 0, -1):
        G[i - 1] = (G[i] @ layers[i][0].T) * sp[i - 1]
    grad = join_params([(acts[i].T @ G[i], G[i].sum(axis=0)) for i in range(L)])
    return Lin(tuple(dims), activation, loss, X, y, layers, acts, sp, out, value, og, G, grad, probs)


def hz_apply(lin: Lin, T):
    """Per-example output Hessian (models.py:199-204)."""
    if lin.loss == "mse":
        return T
    p = lin.probs
    return p * T - p * np.sum(p * T, axis=1, keepdims=True)


def jvp_all(lin: Lin, v):
    """Pre-activation tangents dz[l] and hidden tangents da[l] (models.py:243-272)."""
    tang = split_params(lin.dims, v)
    dzs, das = [], [None]
    da = None
    for i, (W, _) in enumerate(lin.layers):
        dz = lin.acts[i] @ tang[i][0] + tang[i][1]
        if da is not None:
            dz = dz + da @ W
        dzs.append(dz)
        if i < lin.L - 1:
            da = lin.sp[i] * dz
            das.append(da)
    return dzs, das


def jvp(lin: Lin, v):
    """Output tangents J_i v, (b, c) (models.py:243-255)."""
    return jvp_all(lin, v)[0][-1]


def vjp(lin: Lin, U):
    """sum_i J_i^T u_i, no 1/b (models.py:274-285)."""
    parts = [None] * lin.L
    G = np.asarray(U, dtype=np.float64)
    for i in range(lin.L - 1, -1, -1):
        parts[i] = (lin.acts[i].T @ G, G.sum(axis=0))
        if i > 0:
            G = (G @ lin.layers[i][0].T) * lin.sp[i - 1]
    return join_params(parts)


def ggn_matvec(lin: Lin, v):
    """(1/b) J^T H_z J v (curvature.py:109-110)."""
    return vjp(lin, hz_apply(lin, jvp(lin, v))) * (1.0 / lin.b)


def hvp(lin: Lin, v):
    """Exact Hessian-vector product, forward-over-reverse (models.py:287-307)."""
    tang = split_params(lin.dims, v)
    dzs, das = jvp_all(lin, v)
    dG = hz_apply(lin, dzs[-1]) / lin.b
    parts = [None] * lin.L
    for i in range(lin.L - 1, -1, -1):
        gW = lin.acts[i].T @ dG
        if das[i] is not None:
            gW = gW + das[i].T @ lin.G[i]
        parts[i] = (gW, dG.sum(axis=0))
        if i > 0:
            W = lin.layers[i][0]
            nxt = (dG @ W.T + lin.G[i] @ tang[i][0].T) * lin.sp[i - 1]
            if lin.activation == "tanh":  # _sp_second, models.py:192-197
                spp = -2.0 * lin.acts[i] * lin.sp[i - 1]
                nxt = nxt + (lin.G[i] @ W.T) * spp * dzs[i - 1]
            dG = nxt
    return join_params(parts)


def matvec(lin: Lin, kind: str, v):
    return hvp(lin, v) if kind == "hessian" else ggn_matvec(lin, v)


def hz_roots(lin: Lin):
    """Per-example symmetric root / pseudo-inverse root of H_z (models.py:206-239)."""
    if lin.roots is not None:
        return lin.roots
    b, c = lin.out.shape
    if lin.loss == "mse":
        eye = np.broadcast_to(np.eye(c), (b, c, c)).copy()
        lin.roots = (eye, eye)
        return lin.roots
    p = lin.probs
    if not np.all(np.isfinite(p)):
        nan = np.full((b, c, c), np.nan)
        lin.roots = (nan, nan.copy())
        return lin.roots
    H = np.zeros((b, c, c))
    idx = np.arange(c)
    H[:, idx, idx] = p
    H -= p[:, :, None] * p[:, None, :]
    lam, Q = np.linalg.eigh(H)
    keep = lam > 1e-10 * np.maximum(lam.max(axis=1, keepdims=True), 0.0)
    r = np.where(keep, np.sqrt(np.maximum(lam, 0.0)), 0.0)
    ri = np.where(keep, 1.0 / np.where(keep, r, 1.0), 0.0)
    half = (Q * r[:, None, :]) @ np.swapaxes(Q, 1, 2)
    pinv = (Q * ri[:, None, :]) @ np.swapaxes(Q, 1, 2)
    lin.roots = (half, pinv)
    return lin.roots


def row_seeds_rhs(lin: Lin):
    """Row-space seeds and rhs of a GGN snapshot (curvature.py:112-119)."""
    half, pinv = hz_roots(lin)
    if lin.loss == "mse":
        return half, lin.out_grad.ravel().copy()
    return half, np.einsum("bij,bj->bi", pinv, lin.out_grad).ravel()


def output_gram(lin: Lin, seeds):
    """Layer-wise Gram of the seeded Jacobian rows (models.py:309-334)."""
    b, k, c = seeds.shape
    m = b * k
    gram = np.zeros((m, m))
    D = np.asarray(seeds, dtype=np.float64)
    for i in range(lin.L - 1, -1, -1):
        A = lin.acts[i]
        SA = A @ A.T + 1.0
        D2 = D.reshape(m, -1)
        SD = D2 @ D2.T
        gram += SD * np.kron(SA, np.ones((k, k)))
        if i > 0:
            D = (D @ lin.layers[i][0].T) * lin.sp[i - 1][:, None, :]
    return gram


def row_apply(lin: Lin, seeds, v):
    """J_hat v (curvature.py:47-51)."""
    return np.einsum("bij,bj->bi", seeds, jvp(lin, v)).ravel()


def row_transpose(lin: Lin, seeds, u):
    """J_hat^T u (curvature.py:53-60)."""
    U = np.asarray(u, dtype=np.float64).reshape(lin.b, -1)
    return vjp(lin, np.einsum("bij,bj->bi", seeds, U))


# --------------------------------------------------------------------------
# Solvers  (solvers.py:45-174)
# --------------------------------------------------------------------------
DIAG_FLOOR = 1e-12


@dataclass
class CgOut:
    x: np.ndarray
    iterations: int
    converged: bool
    relres: float
    negative_curvature: bool
    gv_count: int


def cg(mv, rhs, lam, tol=1e-5, maxiter=10, stabilise_every=10, precond=None, x0=None,
       floor=DIAG_FLOOR) -> CgOut:
    """Damped (P)CG on raw arrays, reference control flow (solvers.py:60-114).

    `mv` is the undamped operator; lam*x is added here.  gv_count counts the
    operator applications (instrumentation only).
    """
    count = [0]

    def A(x):
        count[0] += 1
        return mv(x) + lam * x

    bnorm = float(np.linalg.norm(rhs))
    if bnorm == 0.0:
        return CgOut(np.zeros_like(rhs), 0, True, 0.0, False, 0)
    minv = None if precond is None else 1.0 / (np.maximum(precond, floor) + lam)
    if x0 is not None and np.any(x0):
        x = np.array(x0, dtype=np.float64)
        r = rhs - A(x)
    else:
        x = np.zeros_like(rhs)
        r = rhs.copy()
    relres = float(np.linalg.norm(r)) / bnorm
    if relres <= tol:
        return CgOut(x, 0, True, relres, False, count[0])
    z = r if minv is None else minv * r
    p = z.copy()
    rz = float(np.dot(r, z))
    for k in range(1, maxiter + 1):
        Ap = A(p)
        pAp = float(np.dot(p, Ap))
        if not math.isfinite(pAp):
            return CgOut(x, k, False, relres, False, count[0])
        if pAp <= 0.0:
            return CgOut(x, k, False, relres, True, count[0])
        alpha = rz / pAp
        step = alpha * p
        if not np.all(np.isfinite(step)):
            return CgOut(x, k, False, relres, False, count[0])
        x = x + step
        if stabilise_every and k % stabilise_every == 0:
            r = rhs - A(x)
        else:
            r = r - alpha * Ap
        relres = float(np.linalg.norm(r)) / bnorm
        if not math.isfinite(relres):
            return CgOut(x, k, False, relres, False, count[0])
        if relres <= tol:
            return CgOut(x, k, True, relres, False, count[0])
        z = r if minv is None else minv * r
        rz_new = float(np.dot(r, z))
        p = z + (rz_new / rz) * p
        rz = rz_new
    return CgOut(x, maxiter, False, relres, False, count[0])


def row_cholesky(gram, rhs, mu):
    """(gram + mu I) v = rhs via LAPACK potrf/potrs (solvers.py:146-161)."""
    A = np.asarray(gram, dtype=np.float64) + mu * np.eye(gram.shape[0])
    try:
        cf = scipy.linalg.cho_factor(A, lower=True, check_finite=False)
    except scipy.linalg.LinAlgError as exc:
        raise ValueError("row system is not positive definite; mu too small or gram invalid") from exc
    return scipy.linalg.cho_solve(cf, rhs, check_finite=False)


# --------------------------------------------------------------------------
# Control + estimators  (control.py:65-127, telemetry.py:91-126)
# --------------------------------------------------------------------------

def rho_of(loss_before, loss_after, g, u, Hu, clip=5.0):
    """Gain ratio with NaN sentinel (control.py:80-102). Returns (pred, rho)."""
    pred = -(float(np.dot(g, u)) + 0.5 * float(np.dot(Hu, u)))
    if not math.isfinite(pred) or pred <= 1e-15:
        return pred, float("nan")
    return pred, float(np.clip((loss_before - loss_after) / pred, -clip, clip))


def tr_update(lam, rho, lower=0.25, upper=0.75, good=0.5, bad=1.5, lo=1e-12, hi=1e6):
    """LM damping update; NaN rho is a no-op (control.py:105-118)."""
    if rho is None or math.isnan(rho):
        return lam
    if rho >= upper:
        lam = lam * good
    elif rho <= lower:
        lam = lam * bad
    return min(max(lam, lo), hi)


def tr_escalate(lam, bad=1.5, lo=1e-12, hi=1e6):  # control.py:121-127
    return min(max(lam * bad, lo), hi)


def hutchinson_diag(mv, rng: ORng, d, n_probes):  # telemetry.py:91-99
    acc = np.zeros(d)
    for _ in range(n_probes):
        z = rademacher(rng, d)
        acc += z * mv(z)
    return acc / n_probes


def hutchinson_trace(mv, rng: ORng, d, n_probes):  # telemetry.py:102-110
    acc = 0.0
    for _ in range(n_probes):
        z = rademacher(rng, d)
        acc += float(np.dot(z, mv(z)))
    return acc / n_probes


def power_iter_top_eig(mv, rng: ORng, d, iters):  # telemetry.py:113-126
    v = rademacher(rng, d) / np.sqrt(d)
    ray = 0.0
    for _ in range(iters):
        hv = mv(v)
        ray = float(np.dot(v, hv))
        nrm = float(np.linalg.norm(hv))
        if nrm == 0.0:
            return 0.0
        v = hv / nrm
    return ray


def ema_diag(diag, new, beta):  # control.py:70-77
    return np.maximum(beta * diag + (1.0 - beta) * new, 0.0)


# --------------------------------------------------------------------------
# Post-direction chain (transforms.py:121-199): every link kind
# --------------------------------------------------------------------------

def schedule_value(kind, t, p):
    """Learning-rate schedules (transforms.py:121-145)."""
    a0 = float(p.get("alpha0", 1.0))
    if kind == "constant":
        return a0
    if kind == "step_decay":
        return a0 * float(p.get("gamma", 0.1)) ** (t // int(p.get("period", 1000)))
    if kind == "cosine_warmup":
        warm, total = int(p.get("warmup", 0)), int(p["total"])
        if warm > 0 and t < warm:
            return a0 * t / warm
        prog = min((t - warm) / max(total - warm, 1), 1.0)
        return 0.5 * a0 * (1.0 + math.cos(math.pi * prog))
    raise ValueError(kind)


def chain_apply(chain, state, direction, w, t, precond_diag=None):
    """Links are (kind, params) pairs, applied left to right (transforms.py:148-199)."""
    x = np.array(direction, dtype=np.float64)
    new = []
    for (kind, p), st in zip(chain, state):
        if kind == "scale":
            x = x * p["value"]
            new.append({})
        elif kind == "scale_by_schedule":
            x = x * schedule_value(p["schedule"], t, p)
            new.append({})
        elif kind == "trace_momentum":
            m = p["beta"] * st["trace"] + x
            x = m.copy()
            new.append({"trace": m})
        elif kind == "add_decayed_weights":
            x = x + p["weight_decay"] * w
            new.append({})
        elif kind == "clip_global_norm":
            n = float(np.linalg.norm(x))
            if n > p["max_norm"] and n > 0.0:
                x = x * (p["max_norm"] / n)
            new.append({})
        elif kind == "scale_by_adam":
            tt = st["t"] + 1
            m = p["b1"] * st["m"] + (1.0 - p["b1"]) * x
            v = p["b2"] * st["v"] + (1.0 - p["b2"]) * (x * x)
            x = (m / (1.0 - p["b1"] ** tt)) / (np.sqrt(v / (1.0 - p["b2"] ** tt)) + p["eps"])
            new.append({"m": m, "v": v, "t": tt})
        elif kind == "sophia_clip":
            den = np.maximum(p["gamma"] * precond_diag, p["eps"])
            x = np.clip(x / den, -1.0, 1.0)
            new.append({})
        else:
            raise NotImplementedError(kind)
    return x, new


def chain_init(chain, d):
    out = []
    for k, _ in chain:
        if k == "trace_momentum":
            out.append({"trace": np.zeros(d)})
        elif k == "scale_by_adam":
            out.append({"m": np.zeros(d), "v": np.zeros(d), "t": 0})
        else:
            out.append({})
    return out


def gnb_diag(lin: Lin, rng: ORng, n_samples: int):
    """Sampled-label squared-gradient GGN diagonal estimate (telemetry.py:129-160)."""
    p = lin.probs
    b, c = p.shape
    cum = np.cumsum(p, axis=1)
    acc = np.zeros(n_params(lin.dims))
    for _ in range(n_samples):
        u = rng.uniform(b)
        labels = np.minimum((u[:, None] > cum).sum(axis=1), c - 1)
        cot = p.copy()
        cot[np.arange(b), labels] -= 1.0
        gh = vjp(lin, cot / b)
        acc += b * (gh * gh)
    return acc / n_samples


def gen_regression(n, d, noise_std, seed, train_frac=0.9):
    """Linear teacher on a gaussian design, 90/10 split (harness/data.py:49-60)."""
    rng = ORng(seed)
    X = rng.normal(n * d).reshape(n, d)
    beta = rng.normal(d)
    y = (X @ beta + rng.normal(n) * noise_std)[:, None]
    ntr = int(n * train_frac)
    return (X[:ntr], y[:ntr]), (X[ntr:], y[ntr:])


# --------------------------------------------------------------------------
# Planned step (method.py:286-409) for the param-lane / row-lane configs
# --------------------------------------------------------------------------
STEP_FIELDS = ("loss_before", "loss_after", "rho", "lam", "grad_norm", "step_norm",
               "solver_iterations", "solver_converged", "final_relative_residual",
               "diag_mean", "trace_estimate", "top_eig_estimate", "step_index")


@dataclass
class OSpec:
    """Flat restatement of MethodSpec for the oracle (method.py:64-134)."""
    curvature: str | None = "ggn_ce"
    solver: str | None = "cg"          # None (identity) | diag | cg | row_cholesky | row_cg
    tol: float = 1e-5
    maxiter: int = 10
    stabilise_every: int = 10
    warm_start: bool = True
    precond: str | None = None         # None | diag_ema
    precond_beta: float = 0.99
    damping: str = "constant"          # constant | trust_region
    lam0: float = 1.0
    tr_every_k: int = 5
    estimator_every_k: int = -1        # fires when >= 1
    estimator_probes: int = 1
    estimator: str = "hutchinson"      # hutchinson | gnb
    rho_every_k: int = -1
    trace_every_k: int = -1
    trace_probes: int = 1
    top_eig_every_k: int = -1
    top_eig_iters: int = 20
    chain: tuple = (("scale", {"value": 1e-3}), ("scale", {"value": -1.0}))


def _fires(k, t):  # telemetry.py:63-78
    return k >= 1 and t % k == 0


@dataclass
class OState:
    lam: float
    diag: np.ndarray
    chain: list
    warm: np.ndarray | None
    t: int
    rng: ORng


def oracle_init(spec: OSpec, d: int, seed: int = 0) -> OState:  # method.py:286-300
    return OState(spec.lam0, np.zeros(d), chain_init(spec.chain, d), None, 0, ORng(seed))


def preset_ospec(name: str) -> OSpec:
    """The presets of method.py:438-552 as flat oracle specs."""
    def soph(g):
        return (("trace_momentum", {"beta": 0.96}), ("sophia_clip", {"gamma": g, "eps": 1e-12}),
                ("add_decayed_weights", {"weight_decay": 1e-4}),
                ("scale_by_schedule", {"schedule": "constant", "alpha0": 0.01}), ("scale", {"value": -1.0}))
    table = {
        "sophia_g": OSpec(curvature="ggn_ce", solver=None, precond="diag_ema", precond_beta=0.99, lam0=0.0,
                          estimator="gnb", estimator_every_k=10, chain=soph(0.05)),
        "sophia_h": OSpec(curvature="hessian", solver=None, precond="diag_ema", precond_beta=0.99, lam0=0.0,
                          estimator="hutchinson", estimator_every_k=10, chain=soph(0.01)),
        "sophia_n": OSpec(curvature="ggn_ce", solver=None, precond="diag_ema", precond_beta=0.99, lam0=0.0,
                          estimator="hutchinson", estimator_every_k=10, chain=soph(0.05)),
        "adahessian": OSpec(curvature="hessian", solver="diag", precond="diag_ema", precond_beta=0.999, lam0=1.0,
                            estimator="hutchinson", estimator_every_k=1,
                            chain=(("trace_momentum", {"beta": 0.9}),
                                   ("scale_by_schedule", {"schedule": "constant", "alpha0": 0.1}),
                                   ("scale", {"value": -1.0}))),
        "sgd": OSpec(curvature=None, solver=None, lam0=0.0,
                     chain=(("scale_by_schedule", {"schedule": "constant", "alpha0": 0.1}), ("scale", {"value": -1.0}))),
        "sgdm": OSpec(curvature=None, solver=None, lam0=0.0,
                      chain=(("trace_momentum", {"beta": 0.9}), ("add_decayed_weights", {"weight_decay": 5e-4}),
                             ("scale_by_schedule", {"schedule": "constant", "alpha0": 0.05}),
                             ("scale", {"value": -1.0}))),
        "adam": OSpec(curvature=None, solver=None, lam0=0.0,
                      chain=(("scale_by_adam", {"b1": 0.9, "b2": 0.999, "eps": 1e-8}),
                             ("scale_by_schedule", {"schedule": "constant", "alpha0": 1e-3}),
                             ("scale", {"value": -1.0}))),
    }
    return table[name]


def oracle_step(spec: OSpec, dims, activation, loss, w, X, y, st: OState, gv_log=None, masks=None):
    """One planned step; returns (w', state', info dict, direction).  method.py:302-389."""
    t = st.t
    rng = st.rng.clone()
    lin = linearize(dims, activation, loss, w, X, y, masks=masks)
    kind = spec.curvature
    mv = lambda v: matvec(lin, kind, v)  # noqa: E731
    g = lin.grad
    info = {k: float("nan") for k in STEP_FIELDS}
    info.update(solver_iterations=-1, solver_converged=-1, step_index=t)
    info.update(loss_before=lin.value, lam=st.lam, grad_norm=float(np.sqrt(np.dot(g, g))))
    tr_on = spec.damping == "trust_region"

    def abort(iters=-1):
        info.update(solver_iterations=iters, solver_converged=-1, step_norm=0.0)
        lam = tr_escalate(st.lam) if tr_on else st.lam
        return w, OState(lam, st.diag, st.chain, None, t + 1, rng), info, None

    if not (math.isfinite(lin.value) and np.all(np.isfinite(g))):
        return abort()
    warm = None
    if spec.solver is None:  # identity lane: the gradient itself (method.py:239-241)
        direction, iters, conv, relres = g.copy(), -1, -1, float("nan")
    elif spec.solver == "diag":  # solve_diag (solvers.py:45-50)
        direction, iters, conv, relres = g / (np.maximum(st.diag, DIAG_FLOOR) + st.lam), -1, -1, float("nan")
    elif spec.solver == "cg":
        x0 = st.warm if (spec.warm_start and st.warm is not None and st.warm.size == g.size) else None
        res = cg(mv, g, st.lam, spec.tol, spec.maxiter, spec.stabilise_every,
                 st.diag if spec.precond else None, x0)
        if gv_log is not None:
            gv_log.append(res.gv_count)
        direction, iters, conv, relres = res.x, res.iterations, int(res.converged), res.relres
        warm = res.x if spec.warm_start else None
    elif spec.solver == "row_cg":  # method.py:270-282 -> row_solve_cg (solvers.py:164-174)
        seeds, rhs = row_seeds_rhs(lin)
        gram = output_gram(lin, seeds)
        x0 = st.warm if (spec.warm_start and st.warm is not None and st.warm.size == rhs.size) else None
        res = cg(lambda u: gram @ u, rhs, float(lin.b) * st.lam, spec.tol, spec.maxiter, spec.stabilise_every,
                 None, x0)
        direction, iters, conv, relres = row_transpose(lin, seeds, res.x), res.iterations, int(res.converged), \
            res.relres
        warm = res.x if spec.warm_start else None
    else:  # row_cholesky (method.py:262-268)
        seeds, rhs = row_seeds_rhs(lin)
        v = row_cholesky(output_gram(lin, seeds), rhs, float(lin.b) * st.lam)
        direction, iters, conv, relres = row_transpose(lin, seeds, v), -1, 1, float("nan")
    update, chain_state = chain_apply(spec.chain, st.chain, direction, w, t, st.diag)
    info.update(solver_iterations=iters, solver_converged=conv)
    if not math.isnan(relres):
        info["final_relative_residual"] = relres
    if not (np.all(np.isfinite(direction)) and np.all(np.isfinite(update))):
        return abort(iters)
    w_next = w + update
    if not np.all(np.isfinite(w_next)):
        return abort(iters)
    info["step_norm"] = float(np.sqrt(np.dot(update, update)))
    rho = None
    tr_fired = tr_on and _fires(spec.tr_every_k, t)
    if _fires(spec.rho_every_k, t) or tr_fired:
        la = loss_value(dims, activation, loss, w_next, X, y)
        _, rho = rho_of(lin.value, la, g, update, mv(update))
        info.update(loss_after=la, rho=rho)
    diag = st.diag
    if _fires(spec.estimator_every_k, t):
        if spec.estimator == "gnb":
            est = gnb_diag(lin, rng, spec.estimator_probes)
        else:
            est = hutchinson_diag(mv, rng, g.size, spec.estimator_probes)
        diag = ema_diag(diag, est, spec.precond_beta) if spec.precond == "diag_ema" else np.maximum(est, 0.0)
        info["diag_mean"] = float(diag.mean())
    if _fires(spec.trace_every_k, t):
        info["trace_estimate"] = hutchinson_trace(mv, rng, g.size, spec.trace_probes)
    if _fires(spec.top_eig_every_k, t):
        info["top_eig_estimate"] = power_iter_top_eig(mv, rng, g.size, spec.top_eig_iters)
    lam = tr_update(st.lam, rho if tr_fired else None) if tr_on else st.lam
    return w_next, OState(lam, diag, chain_state, warm, t + 1, rng), info, direction


# --------------------------------------------------------------------------
# Synthetic data  (harness/data.py:63-90, harness/run.py:174-192)
# --------------------------------------------------------------------------

def gen_classification(n, d, classes, separation, seed, train_frac=0.9):
    rng = ORng(seed)
    means = np.zeros((classes, d))
    for k in range(classes):
        if k < 2 * d:
            means[k, k // 2] = (separation / 2.0) * (1.0 if k % 2 == 0 else -1.0)
        else:
            u = rng.normal(d)
            means[k] = (separation / 2.0) * u / np.linalg.norm(u)
    labels = (np.arange(n) % classes)[rng.permutation(n)]
    X = means[labels] + rng.normal(n * d).reshape(n, d)
    ntr = int(n * train_frac)
    y = labels.astype(np.int64)
    return (X[:ntr], y[:ntr]), (X[ntr:], y[ntr:])


class Batcher:
    """Epoch permutations, fixed batch size (harness/run.py:174-192)."""

    def __init__(self, X, y, bs, rng: ORng):
        self.X, self.y, self.bs, self.rng = X, y, bs, rng
        self.perm = rng.permutation(X.shape[0])
        self.pos = 0

    def next(self):
        n = self.X.shape[0]
        if self.pos + self.bs > n:
            self.perm = self.rng.permutation(n)
            self.pos = 0
        idx = self.perm[self.pos:self.pos + self.bs]
        self.pos += self.bs
        return self.X[idx], self.y[idx]


def synthetic_batch(b, n0, classes, seed=1, loss="ce"):
    """X = Rng(seed).normal(b*n0); y = integers(b, classes) drawn after X."""
    rng = ORng(seed)
    X = rng.normal(b * n0).reshape(b, n0)
    if loss == "ce":
        return X, rng.integers(b, classes)
    return X, rng.normal(b * classes).reshape(b, classes)
