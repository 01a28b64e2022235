"""Damped solves for the three lanes, on the GPU (solvers.py:1-174 of the reference).

`cg_solve` on a snapshot's matvec runs the whole (P)CG loop on the device
(`cv_cg_solve`: fused vector kernels, fp64 scalars, on-device termination, no
host round trip per iteration).  The row-space solves run natively on a
snapshot's or a caller's dense Gram (`cv_row_solve_cg`, `cv_dense_*`); only an
arbitrary user callable runs the recurrence with torch device ops.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ContractError
from .numeric import ParamVector, _is_torch

DIAG_FLOOR = 1e-12


@dataclass(frozen=True)
class CgConfig:
    tol: float = 1e-5
    maxiter: int = 10
    stabilise_every: int = 10  # explicit residual every k iterations; 0 = never
    warm_start: bool = True
    floor: float = DIAG_FLOOR

    def __post_init__(self):
        if self.tol <= 0:
            raise ContractError("cg tol must be positive")
        if self.maxiter < 1:
            raise ContractError("cg maxiter must be >= 1")


@dataclass(frozen=True)
class SolveResult:
    direction: ParamVector
    iterations: int
    converged: bool
    final_relative_residual: float
    negative_curvature: bool = False
    gv_count: int = 0


def solve_diag(diag: ParamVector, g: ParamVector, lam: float, floor: float = DIAG_FLOOR) -> ParamVector:
    """s_i = g_i / (max(diag_i, floor) + lam)  (solvers.py:45-50)."""
    if diag.layout != g.layout:
        raise ContractError("diag and gradient layouts differ")
    if g.on_device:
        return g.like(g.data / (torch.clamp(diag.data, min=floor) + lam))
    return g.like(g.data / (np.maximum(diag.data, floor) + lam))


def damping_to_row(lam: float, b: int) -> float:
    """Row-space damping mu = b * lam under mean reduction (solvers.py:53-57)."""
    if lam < 0 or b < 1:
        raise ContractError("damping_to_row requires lam >= 0 and b >= 1")
    return float(b) * float(lam)


def _snapshot_of(matvec):
    return getattr(matvec, "__self__", None) if getattr(matvec, "__name__", "") == "_matvec" else None


def device_cg(snap, g: torch.Tensor, lam: float, config: CgConfig, precond=None, x0=None, out=None, stats=None):
    """Enqueue the device (P)CG; returns (x, stats_tensor) without synchronising."""
    rt = snap.rt
    x = torch.empty_like(g) if out is None else out
    st = torch.empty(_lib.CG_STATS_BYTES, dtype=torch.uint8, device=rt.device) if stats is None else stats
    rt.bind_stream()
    rt.call("cv_cg_solve", snap.h, snap._kind_code, g.data_ptr(), float(lam), float(config.tol), int(config.maxiter),
            int(config.stabilise_every), _lib.ptr(precond), float(config.floor), _lib.ptr(x0), x.data_ptr(),
            st.data_ptr())
    return x, st


def read_cg_stats(st: torch.Tensor) -> _lib.CgStats:
    raw = st.cpu().numpy().tobytes()
    return _lib.CgStats.from_buffer_copy(raw)


def cg_solve(matvec, g: ParamVector, lam: float, config: CgConfig, precond: ParamVector | None = None,
             x0: ParamVector | None = None) -> SolveResult:
    """Parameter-space (P)CG on a matrix-free operator (solvers.py:117-143)."""
    snap = _snapshot_of(matvec)
    if snap is not None:
        gd = g.data if g.on_device else torch.from_numpy(np.asarray(g.data, dtype=np.float32)).to(snap.rt.device)
        pre = None
        if precond is not None:
            pre = precond.data if precond.on_device else torch.from_numpy(
                np.asarray(precond.data, dtype=np.float32)).to(snap.rt.device)
        xx = None
        if x0 is not None:
            xx = x0.data if x0.on_device else torch.from_numpy(np.asarray(x0.data, dtype=np.float32)).to(snap.rt.device)
        x, st = device_cg(snap, gd.contiguous(), lam, config, pre, xx)
        s = read_cg_stats(st)
        return SolveResult(ParamVector(x, g.layout), int(s.iterations), bool(s.converged), float(s.relres),
                           bool(s.neg_curv), int(s.gv_count))
    x, it, conv, rel, neg, gv = _cg_generic(lambda a: _as_t(matvec(g.like(a)).data, a), _as_t(g.data), lam, config,
                                            None if precond is None else _as_t(precond.data),
                                            None if x0 is None else _as_t(x0.data))
    return SolveResult(g.like(x), it, conv, rel, neg, gv)


def _as_t(a, like=None):
    if _is_torch(a):
        return a
    dev = like.device if like is not None and _is_torch(like) else ("cuda" if torch.cuda.is_available() else "cpu")
    return torch.as_tensor(np.asarray(a), dtype=torch.float64, device=dev)


def _cg_generic(mv, rhs, lam, cfg: CgConfig, precond=None, x0=None):
    """The reference recurrence (solvers.py:60-114) on torch tensors, for operators
    that are not snapshot products (dense Grams, user callables)."""
    gv = 0

    def A(x):
        nonlocal gv
        gv += 1
        return mv(x) + lam * x

    bnorm = float(torch.linalg.vector_norm(rhs.double()))
    if bnorm == 0.0:
        return torch.zeros_like(rhs), 0, True, 0.0, False, 0
    minv = None if precond is None else 1.0 / (torch.clamp(precond, min=cfg.floor) + lam)
    if x0 is not None and bool(torch.any(x0 != 0)):
        x = x0.clone()
        r = rhs - A(x)
    else:
        x = torch.zeros_like(rhs)
        r = rhs.clone()
    relres = float(torch.linalg.vector_norm(r.double())) / bnorm
    if relres <= cfg.tol:
        return x, 0, True, relres, False, gv
    z = r if minv is None else minv * r
    p = z.clone()
    rz = float(torch.dot(r.double(), z.double()))
    for k in range(1, cfg.maxiter + 1):
        ap = A(p)
        pap = float(torch.dot(p.double(), ap.double()))
        if not math.isfinite(pap):
            return x, k, False, relres, False, gv
        if pap <= 0.0:
            return x, k, False, relres, True, gv
        alpha = rz / pap
        step = alpha * p
        if not bool(torch.all(torch.isfinite(step))):
            return x, k, False, relres, False, gv
        x = x + step
        if cfg.stabilise_every and k % cfg.stabilise_every == 0:
            r = rhs - A(x)
        else:
            r = r - alpha * ap
        relres = float(torch.linalg.vector_norm(r.double())) / bnorm
        if not math.isfinite(relres):
            return x, k, False, relres, False, gv
        if relres <= cfg.tol:
            return x, k, True, relres, False, gv
        z = r if minv is None else minv * r
        rz_new = float(torch.dot(r.double(), z.double()))
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, cfg.maxiter, False, relres, False, gv


def _dense_gram(gram, rhs):
    G = _as_t(gram)
    if not G.is_cuda:
        G = G.to("cuda")
    G = G.to(torch.float32).contiguous()
    r = torch.as_tensor(rhs).to(device=G.device, dtype=torch.float32).contiguous().reshape(-1) \
        if _is_torch(rhs) else torch.from_numpy(np.ascontiguousarray(rhs, dtype=np.float32)).to(G.device).reshape(-1)
    if G.dim() != 2 or G.shape[0] != G.shape[1]:
        raise ContractError("gram must be a square matrix")
    if tuple(r.shape) != (G.shape[0],):
        raise ContractError("rhs length does not match gram")
    return G, r


def row_solve_cholesky(gram, rhs, mu: float, row=None):
    """(gram + mu I) v = rhs (solvers.py:146-161), native blocked Cholesky.

    With `row` (a snapshot's RowOps whose Gram this is) the snapshot's resident Gram
    is factored; otherwise the caller's dense Gram (`cv_dense_cholesky_solve`).  A
    not-PD system raises ContractError.
    """
    if row is not None:
        return row.solve_cholesky(mu, rhs)
    from .runtime import runtime

    rt = runtime()
    G, r = _dense_gram(gram, rhs)
    out = torch.empty_like(r)
    rt.bind_stream()
    rt.call("cv_dense_cholesky_solve", rt.h, G.data_ptr(), G.shape[0], float(mu), r.data_ptr(), out.data_ptr())
    return out


def row_solve_cg(gram_matvec, rhs, mu: float, config: CgConfig, x0=None):
    """Row-space CG on (gram + mu I) v = rhs (solvers.py:164-174).

    `gram_matvec` may be a snapshot's `row.gram_matvec`, a dense Gram matrix, or
    `lambda u: gram @ u` over one (the reference's own call, method.py:279: pass the
    matrix to keep the loop on the device); any other callable runs the recurrence
    with device ops that read the scalars back every iteration."""
    from .runtime import runtime

    owner = getattr(gram_matvec, "__self__", None)
    gram = None
    if owner is not None and getattr(gram_matvec, "__name__", "") == "gram_matvec":
        gram = owner.gram()
    elif _is_torch(gram_matvec) or isinstance(gram_matvec, np.ndarray):
        gram = gram_matvec
    if gram is not None:
        rt = runtime()
        G, r = _dense_gram(gram, rhs)
        out = torch.empty_like(r)
        st = torch.empty(_lib.CG_STATS_BYTES, dtype=torch.uint8, device=G.device)
        xx = None if x0 is None else torch.as_tensor(x0).to(device=G.device, dtype=torch.float32).contiguous()
        rt.bind_stream()
        rt.call("cv_dense_cg_solve", rt.h, G.data_ptr(), G.shape[0], float(mu), r.data_ptr(), float(config.tol),
                int(config.maxiter), int(config.stabilise_every), _lib.ptr(xx), out.data_ptr(), st.data_ptr())
        s = read_cg_stats(st)
        return out, int(s.iterations), bool(s.converged), float(s.relres)
    r = _as_t(rhs)
    x, it, conv, rel, _, _ = _cg_generic(lambda u: _as_t(gram_matvec(u), r), r, mu, config,
                                         x0=None if x0 is None else _as_t(x0, r))
    return x, it, conv, rel
