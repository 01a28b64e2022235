"""Per-process device runtime: one native context per (device, world).

One process drives one GPU.  Under `torch.distributed` with world > 1 the context
owns the collectives of the batch-sharded path: every curvature product, gradient
and loss is all-reduced inside the native library.  With an NCCL process group the
library runs its own NCCL communicator (unique id broadcast through the default
group; per-layer gradient all-reduces on a comm stream).  With a gloo process group
(e.g. several ranks sharing one GPU, or CPU-side transport) the library calls back
into `_HostComm`, which stages the buffer through the host and all-reduces it with
the process group -- the same library code path, another transport.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from . import _lib
from .errors import ContractError

_RUNTIMES: dict = {}
_LOCAL = False


class _CudaArray:
    """Zero-copy torch view of a raw device buffer (__cuda_array_interface__)."""

    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None, "stream": None}


class _HostComm:
    """cv_comm_fn over the default torch.distributed group (host-staged all-reduce)."""

    def __init__(self, device):
        self.device = device
        self.calls = 0
        self.fn = _lib.COMM_FN(self._allreduce)  # keep the ctypes thunk alive

    def _allreduce(self, user, dtype, buf, count, stream):
        import torch.distributed as dist

        try:
            torch.cuda.ExternalStream(stream, device=self.device).synchronize() if stream else \
                torch.cuda.synchronize(self.device)
            t = torch.as_tensor(_CudaArray(buf, count, "<f4" if dtype == 0 else "<f8"), device=self.device)
            h = t.cpu()
            dist.all_reduce(h)
            t.copy_(h)
            torch.cuda.synchronize(self.device)
            self.calls += 1
            return 0
        except Exception:  # pragma: no cover - reported to the library as a failed collective
            return 1


class Runtime:
    def __init__(self, device: int = 0, world: int = 1, rank: int = 0, nccl_id: bytes | None = None,
                 host_comm: bool = False):
        if not torch.cuda.is_available():
            raise RuntimeError("curvopt_b200 requires a CUDA device (B200, sm_100a); none is visible")
        self.lib = _lib.lib()
        self.device = torch.device("cuda", device)
        self.world, self.rank = world, rank
        h = C.c_void_p()
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        with torch.cuda.device(self.device):
            rc = self.lib.cv_ctx_create(device, world, rank, idbuf, C.byref(h))
        if rc != 0:
            msg = self.lib.cv_last_error(h) if h.value else b"context creation failed"
            raise _lib.DeviceError((msg or b"").decode())
        self.h = h
        self.comm = None
        if host_comm:
            self.comm = _HostComm(self.device)
            _lib.check(self.lib.cv_ctx_set_comm(self.h, self.comm.fn, None), self.h)
        engine = os.environ.get("CURVOPT_ENGINE", "auto")
        self.set_engine(engine)

    def set_engine(self, name: str) -> None:
        _lib.check(self.lib.cv_ctx_set_engine(self.h, _lib.ENGINE[name]), self.h)

    def bind_stream(self) -> None:
        """Enqueue subsequent native work on torch's current stream."""
        s = torch.cuda.current_stream(self.device)
        self.lib.cv_ctx_set_stream(self.h, C.c_void_p(s.cuda_stream))

    def call(self, name: str, *args) -> None:
        _lib.check(getattr(self.lib, name)(*args), self.h)

    def launches(self) -> int:
        return int(self.lib.cv_kernel_launches(self.h))

    def close(self) -> None:
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.cv_ctx_destroy(self.h)
            self.h = C.c_void_p()


def _dist_info():
    import torch.distributed as dist

    if not _LOCAL and dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank(), dist.get_backend()
    return 1, 0, None


def set_local(on: bool = True) -> None:
    """Replicas: ignore the process group (each rank runs the whole batch on its own GPU,
    no collectives) -- the row lane's multi-GPU mode."""
    global _LOCAL
    _LOCAL = bool(on)


def runtime(device: int | None = None) -> Runtime:
    """The process-wide runtime for `device` (default: current CUDA device)."""
    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    world, rank, backend = _dist_info()
    key = (device, world)
    rt = _RUNTIMES.get(key)
    if rt is None:
        nccl_id = None
        host_comm = world > 1 and backend != "nccl"
        if world > 1 and not host_comm:
            import torch.distributed as dist

            buf = C.create_string_buffer(128)
            if rank == 0:
                lib = _lib.lib()
                if lib.cv_nccl_unique_id(buf) != 0:
                    raise _lib.DeviceError("ncclGetUniqueId failed")
            obj = [bytes(buf.raw) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nccl_id = obj[0]
        rt = Runtime(device, world, rank, nccl_id, host_comm=host_comm)
        _RUNTIMES[key] = rt
    rt.bind_stream()
    return rt


def local_runtime(device: int | None = None) -> Runtime:
    """A world-1 runtime on the same device: work that every rank does whole (the
    distributed row lane's whole-batch snapshot).  Same object as runtime() at world 1."""
    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    key = (device, 1)
    rt = _RUNTIMES.get(key)
    if rt is None:
        rt = Runtime(device, 1, 0)
        _RUNTIMES[key] = rt
    rt.bind_stream()
    return rt


def gather_rows(t: torch.Tensor, row_offset: int, total: int) -> torch.Tensor:
    """The global batch's rows on every rank: each rank's rows [row_offset, row_offset +
    len) placed by offset (torch.distributed all-gather: on the device under NCCL, through
    host memory under gloo).  Raises if the shards do not tile [0, total)."""
    import torch.distributed as dist

    world = dist.get_world_size()
    meta = [None] * world
    dist.all_gather_object(meta, (int(row_offset), int(t.shape[0])))
    spans = sorted(meta)
    pos = 0
    for off, n in spans:
        if off != pos:
            raise ContractError("batch shards do not tile the global batch")
        pos += n
    if pos != total:
        raise ContractError("batch shards do not add up to the global batch size")
    nmax = max(n for _, n in meta)
    pad = torch.zeros((nmax,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    if dist.get_backend() != "nccl":
        pad = pad.cpu()
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    full = torch.empty((total,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    for (off, n), q in zip(meta, parts):
        full[off:off + n] = q[:n].to(t.device)
    return full


def shutdown() -> None:
    for rt in list(_RUNTIMES.values()):
        rt.close()
    _RUNTIMES.clear()
