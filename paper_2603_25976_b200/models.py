"""MLP model description, batches, and the differentiation primitives.

Same model class as curvopt.models (models.py:30-425): dense layers with bias,
relu/tanh hidden activations, linear output, mean MSE (0.5||z-y||^2) or softmax-CE.
The primitives (forward, gradient, JVP, VJP, HVP) run on the GPU through one
device linearization (`curvature.make_snapshot`); nothing here computes on the CPU.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import ContractError
from .numeric import Layout, ParamVector, Rng, _is_torch


@dataclass(frozen=True)
class Model:
    input_dim: int
    hidden_widths: tuple[int, ...]
    output_dim: int
    activation: str = "relu"

    def __post_init__(self):
        object.__setattr__(self, "hidden_widths", tuple(int(h) for h in self.hidden_widths))
        if self.activation not in ("relu", "tanh"):
            raise ContractError(f"unknown activation {self.activation!r}")

    @property
    def dims(self) -> tuple[int, ...]:
        return (self.input_dim, *self.hidden_widths, self.output_dim)

    @property
    def n_layers(self) -> int:
        return len(self.hidden_widths) + 1


@dataclass(frozen=True)
class Batch:
    """Inputs plus targets (float matrix for mse, class indices for ce).

    `global_size` is the batch size the loss mean is taken over; it differs from
    the local row count only for a rank's shard of a data-parallel batch, whose
    first row is row `row_offset` of the global batch (the per-row random streams,
    e.g. gnb_diag's label draws, index the global batch).
    """

    inputs: object
    targets: object
    loss_kind: str
    global_size: int | None = None
    row_offset: int = 0
    _dev: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        X = self.inputs
        if _is_torch(X):
            if X.dim() != 2 or X.shape[0] < 1:
                raise ContractError("batch inputs must be a (b, input_dim) matrix with b >= 1")
        else:
            # float32 host arrays stay float32 (the device precision); anything else
            # is coerced to float64 like the reference Batch (models.py:60)
            X = np.asarray(X) if getattr(X, "dtype", None) == np.float32 else np.asarray(X, dtype=np.float64)
            if X.ndim != 2 or X.shape[0] < 1:
                raise ContractError("batch inputs must be a (b, input_dim) matrix with b >= 1")
            object.__setattr__(self, "inputs", X)
        b = X.shape[0]
        y = self.targets
        if self.loss_kind == "mse":
            if not _is_torch(y):
                y = np.asarray(y, dtype=np.float64)
            if y.ndim == 1:
                y = y[:, None]
            if y.shape[0] != b:
                raise ContractError("targets row count does not match inputs")
        elif self.loss_kind == "ce":
            if _is_torch(y):
                if y.dtype.is_floating_point:
                    raise ContractError("ce targets must be integer class indices")
            else:
                y = np.asarray(y)
                if not np.issubdtype(y.dtype, np.integer):
                    raise ContractError("ce targets must be integer class indices")
            if y.ndim != 1 or y.shape[0] != b:
                raise ContractError("ce targets must be a (b,) index vector")
            # a loader that holds the host copy of the labels passes its minimum in
            # _dev["_ymin"] (no device read, no sync); otherwise read it here
            ymin = self._dev.get("_ymin")
            if (int(y.min()) if ymin is None else ymin) < 0:
                raise ContractError("ce class indices must be non-negative")
        else:
            raise ContractError(f"unknown loss kind {self.loss_kind!r}")
        object.__setattr__(self, "targets", y)
        if self.global_size is None:
            object.__setattr__(self, "global_size", int(b))
        elif self.global_size < b:
            raise ContractError("global_size smaller than the local shard")
        if self.row_offset < 0 or self.row_offset + b > self.global_size:
            raise ContractError("shard rows outside the global batch")

    @property
    def size(self) -> int:
        return int(self.inputs.shape[0])

    def max_label(self) -> int:
        """Largest class index (ce); cached, one device read at most per batch."""
        v = self._dev.get("_ymax")
        if v is None:
            v = int(self.targets.max().item()) if _is_torch(self.targets) else int(self.targets.max())
            self._dev["_ymax"] = v
        return v

    def device_arrays(self, device):
        """(X fp32 [b, n0], y int64 [b] or fp32 [b, c]) on `device`, cached per batch."""
        import torch

        key = str(device)
        hit = self._dev.get(key)
        if hit is not None:
            return hit
        X, y = self.inputs, self.targets
        if _is_torch(X):
            Xd = X.to(device=device, dtype=torch.float32, non_blocking=True).contiguous()
        else:
            Xd = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).pin_memory().to(device, non_blocking=True)
        if self.loss_kind == "ce":
            if _is_torch(y):
                yd = y.to(device=device, dtype=torch.int64, non_blocking=True).contiguous()
            else:
                yd = torch.from_numpy(np.ascontiguousarray(y, dtype=np.int64)).pin_memory().to(device, non_blocking=True)
        else:
            if _is_torch(y):
                yd = y.to(device=device, dtype=torch.float32).contiguous()
            else:
                yd = torch.from_numpy(np.ascontiguousarray(y, dtype=np.float32)).pin_memory().to(device, non_blocking=True)
        self._dev[key] = (Xd, yd)
        return Xd, yd


def param_layout(model: Model) -> Layout:
    """Per layer ("layer{l}.w", (in, out)) then ("layer{l}.b", (out,)) (models.py:87-93)."""
    d = model.dims
    out = []
    for l in range(model.n_layers):
        out += [(f"layer{l}.w", (d[l], d[l + 1])), (f"layer{l}.b", (d[l + 1],))]
    return tuple(out)


def param_count(model: Model) -> int:
    d = model.dims
    return sum((d[l] + 1) * d[l + 1] for l in range(model.n_layers))


def layer_offsets(model: Model) -> list[int]:
    d = model.dims
    offs, o = [], 0
    for l in range(model.n_layers):
        offs.append(o)
        o += (d[l] + 1) * d[l + 1]
    return offs


def init_params(model: Model, rng: Rng) -> ParamVector:
    """Gaussian init, gain sqrt(2) on relu hidden layers, zero biases (models.py:101-112)."""
    d, L = model.dims, model.n_layers
    chunks = []
    for l in range(L):
        gain = math.sqrt(2.0) if (l < L - 1 and model.activation == "relu") else 1.0
        chunks.append(rng.normal(d[l] * d[l + 1]) * (gain / math.sqrt(d[l])))
        chunks.append(np.zeros(d[l + 1]))
    return ParamVector(np.concatenate(chunks), param_layout(model))


def check_layout(model: Model, w: ParamVector) -> None:
    if w.layout != param_layout(model):
        raise ContractError("parameter layout does not match model")


# --- device primitives (each builds one linearization) ----------------------

def linearize(model: Model, w: ParamVector, batch: Batch):
    """Device linearization handle (models.py:337-396); see curvature.Snapshot."""
    from .curvature import build_snapshot

    return build_snapshot(None, model, w, batch)


def forward(model: Model, w: ParamVector, X) -> np.ndarray:
    """Network outputs (b, c) (models.py:143-156)."""
    Xa = X if _is_torch(X) else np.asarray(X, dtype=np.float64)
    if Xa.ndim != 2 or Xa.shape[1] != model.input_dim:
        raise ContractError("input matrix shape does not match model input_dim")
    b = Xa.shape[0]
    if model.output_dim >= 2:
        batch = Batch(Xa, np.zeros(b, dtype=np.int64), "ce")
    else:
        batch = Batch(Xa, np.zeros((b, model.output_dim)), "mse")
    lin = linearize(model, w, batch)
    return lin.outputs()


def loss_value(model: Model, w: ParamVector, batch: Batch) -> float:
    return linearize(model, w, batch).loss_before


def loss_and_grad(model: Model, w: ParamVector, batch: Batch):
    lin = linearize(model, w, batch)
    return lin.loss_before, lin.grad


def hvp(model: Model, w: ParamVector, batch: Batch, v: ParamVector) -> ParamVector:
    return linearize(model, w, batch).hvp(v)


def jvp_outputs(model: Model, w: ParamVector, batch: Batch, v: ParamVector):
    return linearize(model, w, batch).jvp(v)


def vjp_outputs(model: Model, w: ParamVector, batch: Batch, U) -> ParamVector:
    return linearize(model, w, batch).vjp(U)
