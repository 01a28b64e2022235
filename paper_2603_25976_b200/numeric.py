"""Flat parameter vectors with layout metadata, and the SplitMix64 counter RNG.

Mirrors curvopt.numeric (numeric.py:30-162) with one extension: a ParamVector's
`data` may be a host float64 numpy array (the reference's representation) or a
device float32 torch tensor (the B200 representation).  Arithmetic stays on
whichever side the operands live; mixing sides is a ContractError.
"""

from __future__ import annotations

import functools
import math
from dataclasses import dataclass
from typing import Any

import numpy as np

from .errors import ContractError

Layout = tuple[tuple[str, tuple[int, ...]], ...]


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


@functools.lru_cache(maxsize=256)
def _layout_size(layout: Layout) -> int:
    return int(sum(math.prod(int(n) for n in shape) for _, shape in layout))


def layout_size(layout: Layout) -> int:
    """Total element count of a layout (cached: every ParamVector validates against it)."""
    try:
        return _layout_size(layout)
    except TypeError:  # unhashable (list-based) layout
        return int(sum(math.prod(int(n) for n in shape) for _, shape in layout))


@dataclass(frozen=True)
class ParamVector:
    """Flat vector + ordered (name, shape) layout (numeric.py:30-78)."""

    data: Any
    layout: Layout

    def __post_init__(self):
        d = self.data
        if _is_torch(d):
            if d.dim() != 1:
                d = d.reshape(-1)
            if not d.is_contiguous():
                d = d.contiguous()
            n = d.numel()
        else:
            # host: float64 like the reference (numeric.py:41-45); float32 is kept as is
            d = (np.asarray(d) if getattr(d, "dtype", None) == np.float32 else np.asarray(d, dtype=np.float64)).reshape(-1)
            n = d.size
        object.__setattr__(self, "data", d)
        if n != layout_size(self.layout):
            raise ContractError(f"data length {n} does not match layout size {layout_size(self.layout)}")

    @property
    def dim(self) -> int:
        return int(self.data.numel() if _is_torch(self.data) else self.data.size)

    @property
    def on_device(self) -> bool:
        return _is_torch(self.data) and self.data.is_cuda

    def like(self, data) -> "ParamVector":
        return ParamVector(data, self.layout)

    def _check(self, other: "ParamVector") -> None:
        if self.layout != other.layout:
            raise ContractError("layout mismatch between ParamVectors")
        if self.on_device != other.on_device:
            raise ContractError("ParamVectors live on different devices")

    def __add__(self, other):
        self._check(other)
        return self.like(self.data + other.data)

    def __sub__(self, other):
        self._check(other)
        return self.like(self.data - other.data)

    def __mul__(self, scalar):
        return self.like(self.data * float(scalar))

    __rmul__ = __mul__

    def __neg__(self):
        return self.like(-self.data)

    # -- host/device movement -------------------------------------------------
    def to_device(self, device=None) -> "ParamVector":
        if self.on_device:
            return self
        import torch

        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        if _is_torch(self.data):  # host torch tensor (pinned for async copies)
            return self.like(self.data.to(device=dev, dtype=torch.float32, non_blocking=True))
        t = torch.from_numpy(np.ascontiguousarray(self.data, dtype=np.float32))
        return self.like(t.to(dev))

    def to_host(self, like: "ParamVector | None" = None) -> "ParamVector":
        """Device -> host as float32 (numpy, or a torch CPU tensor when `like` is one)."""
        if not self.on_device:
            return self
        if like is not None and _is_torch(like.data):
            import torch

            host = torch.empty(self.data.shape, dtype=self.data.dtype, pin_memory=True)  # caching host allocator
            host.copy_(self.data)
            return self.like(host)
        return self.like(self.data.detach().cpu().numpy())

    def numpy(self) -> np.ndarray:
        return self.to_host().data


def zeros(layout: Layout, like: ParamVector | None = None) -> ParamVector:
    if like is not None and like.on_device:
        import torch

        return ParamVector(torch.zeros(layout_size(layout), dtype=torch.float32, device=like.data.device), layout)
    return ParamVector(np.zeros(layout_size(layout)), layout)


def dot(a: ParamVector, b: ParamVector) -> float:
    a._check(b)
    if a.on_device:
        return float((a.data.double() @ b.data.double()).item())
    return float(np.dot(a.data, b.data))


def global_norm(a: ParamVector) -> float:
    if a.on_device:
        x = a.data.double()
        return float(x.dot(x).sqrt().item())
    return float(np.sqrt(np.dot(a.data, a.data)))


# ---------------------------------------------------------------------------
# SplitMix64 counter stream (numeric.py:95-154): value i = mix(seed + G*(ctr+i)),
# i = 1..n; bit-exact with the reference on every platform.
# ---------------------------------------------------------------------------
_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)
_M64 = 0xFFFFFFFFFFFFFFFF


def _splitmix(seed: int, first: int, n: int) -> np.ndarray:
    k = np.arange(first, first + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + _GAMMA * k
        z ^= z >> np.uint64(30)
        z *= _C1
        z ^= z >> np.uint64(27)
        z *= _C2
        z ^= z >> np.uint64(31)
    return z


class Rng:
    """Counter-based generator; identical (seed, counter) -> identical stream."""

    __slots__ = ("seed", "counter")

    def __init__(self, seed: int, counter: int = 0):
        self.seed = int(seed) & _M64
        self.counter = int(counter)

    def clone(self) -> "Rng":
        return Rng(self.seed, self.counter)

    def _raw(self, n: int) -> np.ndarray:
        out = _splitmix(self.seed, self.counter + 1, n)
        self.counter += n
        return out

    def advance(self, n: int) -> int:
        """Consume n draws without materialising them; returns the old counter."""
        c = self.counter
        self.counter += int(n)
        return c

    def uniform(self, n: int) -> np.ndarray:
        return (self._raw(n) >> np.uint64(11)).astype(np.float64) * 2.0**-53

    def normal(self, n: int) -> np.ndarray:
        half = (n + 1) // 2
        u = self._raw(2 * half)
        u1 = ((u[:half] >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0**-53
        u2 = (u[half:] >> np.uint64(11)).astype(np.float64) * 2.0**-53
        rad = np.sqrt(-2.0 * np.log(u1))
        th = 2 * np.pi * u2
        return np.concatenate([rad * np.cos(th), rad * np.sin(th)])[:n]

    def integers(self, n: int, bound: int) -> np.ndarray:
        return np.minimum((self.uniform(n) * bound).astype(np.int64), bound - 1)

    def permutation(self, n: int) -> np.ndarray:
        return np.argsort(self.uniform(n), kind="stable")

    def split(self) -> "Rng":
        return Rng(int(self._raw(1)[0]), 0)


def rademacher(rng: Rng, n: int) -> np.ndarray:
    """Host +-1 probe (numeric.py:157-162)."""
    if n < 1:
        raise ContractError("rademacher requires n >= 1")
    return (rng._raw(n) >> np.uint64(63)).astype(np.float64) * 2.0 - 1.0


def device_rademacher(rng: Rng, n: int, device=None):
    """The same probe generated on the GPU (fp32 torch tensor); advances rng by n."""
    import torch

    from .runtime import runtime

    if n < 1:
        raise ContractError("rademacher requires n >= 1")
    rt = runtime(None if device is None else torch.device(device).index)
    out = torch.empty(n, dtype=torch.float32, device=rt.device)
    ctr = rng.advance(n)
    rt.call("cv_rademacher", rt.h, rng.seed, ctr, n, out.data_ptr())
    return out
