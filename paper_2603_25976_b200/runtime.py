"""Per-process device runtime: one native context per (device, world).

One process drives one GPU.  Under `torch.distributed` with world > 1 the
context owns an NCCL communicator (unique id broadcast through the default
process group), and every curvature product / gradient / loss is all-reduced
inside the native library.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from . import _lib

_RUNTIMES: dict = {}


class Runtime:
    def __init__(self, device: int = 0, world: int = 1, rank: int = 0, nccl_id: bytes | None = None):
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

    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def runtime(device: int | None = None) -> Runtime:
    """The process-wide runtime for `device` (default: current CUDA device)."""
    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    world, rank = _dist_info()
    key = (device, world)
    rt = _RUNTIMES.get(key)
    if rt is None:
        nccl_id = None
        if world > 1:
            import torch.distributed as dist

            buf = C.create_string_buffer(128)
            if rank == 0:
                lib = _lib.lib()
                if lib.cv_nccl_unique_id(buf) != 0:
                    raise _lib.DeviceError("ncclGetUniqueId failed")
            obj = [bytes(buf.raw) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nccl_id = obj[0]
        rt = Runtime(device, world, rank, nccl_id)
        _RUNTIMES[key] = rt
    rt.bind_stream()
    return rt


def shutdown() -> None:
    for rt in list(_RUNTIMES.values()):
        rt.close()
    _RUNTIMES.clear()
