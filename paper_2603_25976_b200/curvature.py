"""Step-local curvature snapshots on the GPU (curvature.py:1-155 of the reference).

A snapshot is one device linearization (forward, loss, primal backward, gradient)
held by the native library.  Its `matvec` is the undamped GGN product
(1/b) J^T H_z J v or the exact Hessian product, computed by the sm_100a kernels;
`row` exposes the row-space primitives (seeds, rhs, Gram, backprojection).
Exactly one snapshot is built per optimizer step (counter below, as in the
reference's test instrumentation, curvature.py:24-29).
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np
import torch

from . import _lib
from .errors import ContractError
from .models import Batch, Model, check_layout, param_count, param_layout
from .numeric import ParamVector, _is_torch
from .runtime import gather_rows, local_runtime, runtime

CURVATURE_KINDS = ("hessian", "ggn_mse", "ggn_ce")

_snapshot_builds = 0


def snapshot_build_count() -> int:
    return _snapshot_builds


def _device_vec(rt, v: ParamVector):
    if v.on_device:
        t = v.data
        if t.dtype != torch.float32 or t.device != rt.device:
            t = t.to(device=rt.device, dtype=torch.float32)
        return t.contiguous()
    return torch.from_numpy(np.ascontiguousarray(v.data, dtype=np.float32)).to(rt.device)


class RowOps:
    """Row-space primitives of a GGN snapshot (curvature.py:32-65)."""

    def __init__(self, snap: "Snapshot"):
        # weak: a strong back-reference would make every snapshot a GC cycle and keep
        # its device buffers alive until the next collection
        self._snap = weakref.proxy(snap)
        self.m = snap.batch_local * snap.model.output_dim
        self._rhs = None
        self._gram = None
        self._whole = None
        if snap.rt.world > 1:  # the row system is the global batch's (m = b_global * c)
            self.m = snap.batch_size * snap.model.output_dim

    # -- distributed row lane (world > 1) -------------------------------------
    # The row system couples every example of the global batch.  Each rank gathers the
    # batch and builds a whole-batch snapshot on a world-1 context of its GPU (the D
    # chain, seeds and back-projection are done whole, identically on every rank); the
    # Gram and its factorization are distributed over the ranks by
    # cv_row_solve_cholesky_dist / cv_row_solve_cg_dist (block-cyclic row panels; the
    # row vectors are whole and replicated).
    def _whole_snap(self):
        if self._whole is None:
            s = self._snap
            b = s._batch
            X, y = b.device_arrays(s.rt.device)
            Xf = gather_rows(X, b.row_offset, s.batch_size)
            yf = gather_rows(y, b.row_offset, s.batch_size)
            full = Batch(Xf, yf, b.loss_kind, global_size=s.batch_size, row_offset=0)
            self._whole = Snapshot(s.kind, s.model, ParamVector(s.w_dev, s.layout), full, local_runtime(s.rt.device.index),
                                   grad=False)
            s.rt.bind_stream()
        return self._whole

    @property
    def distributed(self) -> bool:
        return self._snap.rt.world > 1

    @property
    def rhs(self):
        if self.distributed:
            return self._whole_snap().row.rhs
        if self._rhs is None:
            s = self._snap
            out = torch.empty(self.m, dtype=torch.float32, device=s.rt.device)
            s.rt.bind_stream()
            s.rt.call("cv_row_rhs", s.h, out.data_ptr())
            self._rhs = out
        return self._rhs

    def gram(self):
        if self.distributed:
            return self._whole_snap().row.gram()
        if self._gram is None:
            s = self._snap
            out = torch.empty((self.m, self.m), dtype=torch.float32, device=s.rt.device)
            s.rt.bind_stream()
            s.rt.call("cv_row_gram", s.h, out.data_ptr())
            self._gram = out
        return self._gram

    def solve_cholesky(self, mu: float, rhs=None):
        """(Gram + mu I) v = rhs on the device (solvers.py:146-161); distributed over
        the ranks at world > 1."""
        s = self._snap
        r = self.rhs if rhs is None else torch.as_tensor(rhs, dtype=torch.float32, device=s.rt.device).contiguous()
        if r.numel() != self.m:
            raise ContractError("rhs length does not match gram")
        out = torch.empty(self.m, dtype=torch.float32, device=s.rt.device)
        s.rt.bind_stream()
        if self.distributed:
            s.rt.call("cv_row_solve_cholesky_dist", s.rt.h, self._whole_snap().h, float(mu), r.data_ptr(),
                      out.data_ptr())
        else:
            s.rt.call("cv_row_solve_cholesky", s.h, float(mu), r.data_ptr(), out.data_ptr())
        return out

    def gram_matvec(self, u):
        """`gram @ u` (method.py:279) on the device."""
        s = self._snap
        u = torch.as_tensor(u, dtype=torch.float32, device=s.rt.device).contiguous().reshape(-1)
        return self.gram() @ u

    def solve_cg(self, mu: float, config, x0=None, stats=None):
        """Row-space CG on (Gram + mu I) v = rhs (solvers.py:164-174), device resident.

        Returns (v, stats) without synchronising; `stats` is a cv_cg_stats buffer."""
        s = self._snap
        if self.distributed:  # Gram products from the ranks' strips
            w = self._whole_snap()
            out = torch.empty(self.m, dtype=torch.float32, device=s.rt.device)
            st = torch.empty(_lib.CG_STATS_BYTES, dtype=torch.uint8, device=s.rt.device) if stats is None else stats
            xx = None if x0 is None else torch.as_tensor(x0, dtype=torch.float32, device=s.rt.device).contiguous()
            s.rt.bind_stream()
            s.rt.call("cv_row_solve_cg_dist", s.rt.h, w.h, float(mu), w.row.rhs.data_ptr(), float(config.tol),
                      int(config.maxiter), int(config.stabilise_every), _lib.ptr(xx), out.data_ptr(), st.data_ptr())
            return out, st
        out = torch.empty(self.m, dtype=torch.float32, device=s.rt.device)
        st = torch.empty(_lib.CG_STATS_BYTES, dtype=torch.uint8, device=s.rt.device) if stats is None else stats
        xx = None
        if x0 is not None:
            xx = torch.as_tensor(x0, dtype=torch.float32, device=s.rt.device).contiguous()
        s.rt.bind_stream()
        s.rt.call("cv_row_solve_cg", s.h, float(mu), self.rhs.data_ptr(), float(config.tol), int(config.maxiter),
                  int(config.stabilise_every), _lib.ptr(xx), out.data_ptr(), st.data_ptr())
        return out, st

    def scaled_row_transpose(self, u) -> ParamVector:
        if self.distributed:
            return self._whole_snap().row.scaled_row_transpose(u)
        s = self._snap
        u = torch.as_tensor(u, dtype=torch.float32, device=s.rt.device).contiguous().reshape(-1)
        if u.numel() != self.m:
            raise ContractError(f"row vector has length {tuple(u.shape)}, expected ({self.m},)")
        out = torch.empty(s.d, dtype=torch.float32, device=s.rt.device)
        s.rt.bind_stream()
        s.rt.call("cv_backproject", s.h, u.data_ptr(), out.data_ptr())
        return ParamVector(out, s.layout)


class Snapshot:
    """Loss, gradient and curvature closures of one (w, batch) point."""

    def __init__(self, kind, model: Model, w: ParamVector, batch: Batch, rt, grad: bool = True):
        self.kind = kind
        self.model = model
        self.rt = rt
        self.layout = param_layout(model)
        self.batch_size = int(batch.global_size)
        self.batch_local = batch.size
        self._batch = batch
        X, y = batch.device_arrays(rt.device)
        if X.shape[1] != model.input_dim:
            raise ContractError("batch input width does not match model input_dim")
        if batch.loss_kind == "ce":
            if model.output_dim < 2:
                raise ContractError("ce loss requires output_dim >= 2")
            if batch.max_label() >= model.output_dim:
                raise ContractError("ce class index out of range")
        elif tuple(y.shape) != (batch.size, model.output_dim):
            raise ContractError("mse targets shape does not match model outputs")
        self.d = param_count(model)
        wd = _device_vec(rt, w)
        self.w_dev = wd
        self._loss = torch.empty(1, dtype=torch.float64, device=rt.device)
        self._grad = torch.empty(self.d, dtype=torch.float32, device=rt.device) if grad else None
        dims = (C.c_int * (model.n_layers + 1))(*model.dims)
        h = C.c_void_p()
        rt.bind_stream()
        rt.call("cv_linearize", rt.h, model.n_layers, dims, _lib.ACT[model.activation], _lib.LOSS[batch.loss_kind],
                wd.data_ptr(), X.data_ptr(), y.data_ptr(), batch.size, self.batch_size, C.byref(h),
                self._loss.data_ptr(), None if self._grad is None else self._grad.data_ptr())
        self.h = h
        self._kind_code = _lib.KIND_HESSIAN if kind == "hessian" else _lib.KIND_GGN
        self.row = RowOps(self) if kind in ("ggn_mse", "ggn_ce") else None
        self._loss_host = None

    # -- scalar / vector state ---------------------------------------------
    @property
    def loss_dev(self):
        return self._loss

    @property
    def loss_before(self) -> float:
        if self._loss_host is None:
            self._loss_host = float(self._loss.item())
        return self._loss_host

    @property
    def grad(self) -> ParamVector:
        return ParamVector(self._grad, self.layout)

    @property
    def matvec(self):
        if self.kind is None:
            return None
        return self._matvec

    def _matvec(self, v: ParamVector) -> ParamVector:
        out = self.apply(self._kind_code, _device_vec(self.rt, v))
        return ParamVector(out, self.layout)

    def apply(self, kind_code: int, v: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if v.numel() != self.d:
            raise ContractError("layout mismatch between ParamVectors")
        out = torch.empty(self.d, dtype=torch.float32, device=self.rt.device) if out is None else out
        self.rt.bind_stream()
        self.rt.call("cv_matvec", self.h, kind_code, v.data_ptr(), out.data_ptr())
        return out

    def hvp(self, v: ParamVector) -> ParamVector:
        return ParamVector(self.apply(_lib.KIND_HESSIAN, _device_vec(self.rt, v)), self.layout)

    def ggn(self, v: ParamVector) -> ParamVector:
        return ParamVector(self.apply(_lib.KIND_GGN, _device_vec(self.rt, v)), self.layout)

    def jvp(self, v: ParamVector):
        vv = _device_vec(self.rt, v)
        out = torch.empty((self.batch_local, self.model.output_dim), dtype=torch.float32, device=self.rt.device)
        self.rt.bind_stream()
        self.rt.call("cv_jvp", self.h, vv.data_ptr(), out.data_ptr())
        return out

    def vjp(self, U) -> ParamVector:
        Ut = U if _is_torch(U) else torch.from_numpy(np.ascontiguousarray(U, dtype=np.float32))
        Ut = Ut.to(device=self.rt.device, dtype=torch.float32).contiguous()
        if tuple(Ut.shape) != (self.batch_local, self.model.output_dim):
            raise ContractError("cotangent matrix shape does not match outputs")
        out = torch.empty(self.d, dtype=torch.float32, device=self.rt.device)
        self.rt.bind_stream()
        self.rt.call("cv_vjp", self.h, Ut.data_ptr(), out.data_ptr())
        return ParamVector(out, self.layout)

    def outputs(self):
        out = torch.empty((self.batch_local, self.model.output_dim), dtype=torch.float32, device=self.rt.device)
        self.rt.bind_stream()
        self.rt.call("cv_snap_outputs", self.h, out.data_ptr())
        return out

    def activation(self, layer: int):
        """Hidden activation a_layer (b x n_layer) as stored on the device (fp32)."""
        out = torch.empty((self.batch_local, self.model.dims[layer]), dtype=torch.float32, device=self.rt.device)
        self.rt.bind_stream()
        self.rt.call("cv_snap_activation", self.h, int(layer), out.data_ptr())
        return out

    def loss_at_dev(self, w: torch.Tensor, out: torch.Tensor) -> None:
        self.rt.bind_stream()
        self.rt.call("cv_loss_at", self.h, w.data_ptr(), out.data_ptr())

    def loss_at(self, w: ParamVector) -> float:
        """Batch loss at another point, same batch, forward only (curvature.py:82-84)."""
        check_layout(self.model, w)
        out = torch.empty(1, dtype=torch.float64, device=self.rt.device)
        self.loss_at_dev(_device_vec(self.rt, w), out)
        return float(out.item())

    def close(self) -> None:
        if getattr(self, "h", None) is not None and self.h.value:
            _lib.lib().cv_snap_free(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_snapshot(kind, model: Model, w: ParamVector, batch: Batch, grad: bool = True) -> Snapshot:
    check_layout(model, w)
    return Snapshot(kind, model, w, batch, runtime(), grad=grad)


def make_snapshot(kind: str | None, model: Model, w: ParamVector, batch: Batch) -> Snapshot:
    """The step's single curvature snapshot (curvature.py:87-131)."""
    global _snapshot_builds
    if kind is not None and kind not in CURVATURE_KINDS:
        raise ContractError(f"unknown curvature kind {kind!r}")
    if kind == "ggn_mse" and batch.loss_kind != "mse":
        raise ContractError("ggn_mse curvature requires an mse batch")
    if kind == "ggn_ce" and batch.loss_kind != "ce":
        raise ContractError("ggn_ce curvature requires a ce batch")
    snap = build_snapshot(kind, model, w, batch)
    _snapshot_builds += 1
    return snap


def hessian_matvec(snapshot: Snapshot, v: ParamVector) -> ParamVector:
    if snapshot.kind != "hessian":
        raise ContractError("hessian_matvec requires a hessian snapshot")
    return snapshot.matvec(v)


def ggn_matvec(snapshot: Snapshot, v: ParamVector) -> ParamVector:
    if snapshot.kind not in ("ggn_mse", "ggn_ce"):
        raise ContractError("ggn_matvec requires a GGN snapshot")
    return snapshot.matvec(v)


def row_gram(snapshot: Snapshot):
    if snapshot.row is None:
        raise ContractError("row primitives are only available for GGN snapshots")
    return snapshot.row.gram()


def backproject(snapshot: Snapshot, v_row) -> ParamVector:
    if snapshot.row is None:
        raise ContractError("row primitives are only available for GGN snapshots")
    return snapshot.row.scaled_row_transpose(v_row)
